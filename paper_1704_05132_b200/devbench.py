"""Measurement helpers for bench.py (device peaks and the end-to-end leg)."""

import ctypes
import time

import numpy as np


def int32_peak_ops():
    """Measured INT32 op/s of the current GPU (rl_int_peak microbenchmark)."""
    from . import _native
    out = np.zeros(1, np.float64)
    _native.check(_native.load().rl_int_peak(_native.ptr(out)), "rl_int_peak")
    return float(out[0])


def _pinned(torch, a):
    t = torch.empty(a.shape, dtype={np.int64: torch.int64, np.uint8: torch.uint8,
                                    np.bool_: torch.uint8}[a.dtype.type], pin_memory=True)
    arr = t.numpy()
    arr[...] = a
    return t, arr


def e2e_steps(torch, _native, dev, shard, steps, world, dist, coll="cuda", pipelined=True):
    """Time `steps` end-to-end descents through the C ABI with pinned host
    buffers: each step uploads the instance and the start plan, runs the VND
    and reads back the final plan, trace and stats -- one rl_vnd_host call
    (uploads chunked and overlapped with the descent) or, pipelined=False,
    rl_instance_update + rl_vnd.  Returns (max-over-ranks total ms, h2d
    bytes, d2h bytes) for the whole job."""
    lib = _native.load()
    keep = []
    arrays = []
    for a in shard.arrays():
        t, arr = _pinned(torch, np.ascontiguousarray(a, np.int64))
        keep.append(t)
        arrays.append(arr)
    sm0, sr0 = dev.initial_solution()
    tm, sm = _pinned(torch, sm0.view(np.uint8))
    tr_, sr = _pinned(torch, sr0.view(np.uint8))
    to, om = _pinned(torch, np.zeros_like(sm))
    tq, orr = _pinned(torch, np.zeros_like(sr))
    keep += [tm, tr_, to, tq]
    trace = np.empty(1 << 16, np.int64)
    nt = np.zeros(1, np.int64)
    st = np.zeros(9, np.int64)
    P = _native.ptr

    def one():
        if pipelined:
            _native.check(lib.rl_vnd_host(dev.h, 4, *[P(a) for a in arrays], P(sm), P(sr), P(om),
                                          P(orr), P(trace), len(trace), P(nt), P(st)),
                          "rl_vnd_host")
            return
        _native.check(lib.rl_instance_update(dev.h, *[P(a) for a in arrays]),
                      "rl_instance_update")
        _native.check(lib.rl_vnd(dev.h, 4, P(sm), P(sr), P(om), P(orr), P(trace), len(trace),
                                 P(nt), P(st)), "rl_vnd")

    one()   # warm
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    h2d = sum(a.nbytes for a in arrays) + sm.nbytes + sr.nbytes
    d2h = om.nbytes + orr.nbytes + int(nt[0]) * 8 + st.nbytes + 24
    tot = torch.tensor([ms, 0.0], dtype=torch.float64, device=coll)
    byt = torch.tensor([h2d, d2h], dtype=torch.int64, device=coll)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        dist.all_reduce(byt, op=dist.ReduceOp.SUM)
    return float(tot[0]), int(byt[0]), int(byt[1])


def other_configs(torch):
    """Secondary BASELINE configs measured on this GPU (reported beside the
    headline; each parity-checked where a reference golden exists):
      c2_vnd  K=1000 T=52 VND to local optimum (ms; golden cost 4,484,593,955)
      c2_gvns K=1000 T=52 full GVNS, W=2, k_max=5: rounds/s over 400 rounds
      c2_gvns_20k  the same over 20,000 rounds (speculative batches pay late)
      c4_vnd  K=10000 T=520 VND to local optimum (ms)
      c5_gvns K=1000 T=52, W=128 workers (one GPU's share of 1,024): rounds/s
    Times are device-synchronised wall clock around the C ABI calls."""
    from . import _native
    from .gvns import SolverConfig, gvns
    from .model import GeneratorConfig, generate_instance

    out = {}

    def vnd_ms(K, T, reps=3):
        inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=0))
        dev = _native.device_instance(inst)
        sm, sr = dev.initial_solution()
        dev.vnd(sm, sr)
        best, st = None, None
        for _ in range(reps):
            _, _, _, st = dev.vnd(sm, sr)
            ms = st["kernel_ns"] / 1e6
            best = ms if best is None else min(best, ms)
        return inst, best, st

    inst2, ms, st = vnd_ms(1000, 52)
    out["c2_vnd"] = {"kernel_ms": ms, "cost": st["cost"], "bit_exact": st["cost"] == 4484593955,
                     "evals_reference": st["evals_reference"]}
    for name, W, R in (("c2_gvns", 2, 400), ("c2_gvns_20k", 2, 20000),
                       ("c5_gvns_1gpu_share", 128, 40)):
        cfg = SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=W, seed=0, max_rounds=R)
        gvns(inst2, SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=W, seed=0,
                                 max_rounds=2))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = gvns(inst2, cfg)
        dt = time.perf_counter() - t0
        out[name] = {"workers": W, "rounds": res.rounds, "seconds": dt,
                     "rounds_per_s": res.rounds / dt, "shakes_per_s": res.shake_calls / dt,
                     "best_cost": res.cost}
    _, ms, st = vnd_ms(10000, 520, reps=2)
    out["c4_vnd"] = {"kernel_ms": ms, "cost": st["cost"], "sweeps": st["sweeps"],
                     "evals_reference": st["evals_reference"],
                     "reference_equiv_evals_per_s": st["evals_reference"] / (ms / 1e3)}
    return out
