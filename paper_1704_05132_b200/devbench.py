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


def _golden(name):
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "tests", "golden", name)
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def _plan_sha(sm, sr):
    import hashlib
    h = hashlib.sha256()
    h.update(np.packbits(np.asarray(sm, bool)).tobytes())
    h.update(np.packbits(np.asarray(sr, bool)).tobytes())
    return h.hexdigest()


def other_configs(torch, clocks=None, roofline=None):
    """Secondary BASELINE configs measured on this GPU (reported beside the
    headline; each parity-checked against a committed golden of the live
    reference / the pinned oracle where one exists):
      c2_vnd      K=1000 T=52 VND to local optimum (golden cost 4,484,593,955)
      c3_int64    C3 on the general int64-value / int64-cost path (variant 16)
      c4_vnd      K=10000 T=520 VND to local optimum (golden: full oracle
                  descent, tests/golden/c4_full.json)
      c2_gvns     K=1000 T=52 full GVNS, W=2, k_max=5: rounds/s over 400 rounds
      c2_gvns_20k the same over 20,000 rounds (speculative batches pay late)
      c5_*        K=1000 T=52 multi-start replicas: W=128 (one GPU's share of
                  8) and all W=1,024 on this GPU: rounds/s, and the
                  round-capped live-reference goldens W=128 x 4, W=1,024 x 2
    VND times are the CUDA-event kernel times of the descent; GVNS times are
    wall clock around gvns() (device-synchronised).  ``roofline(wl,
    kernel_ms)`` adds the issue-slot roofline of a captured workload."""
    from . import _native
    from .gvns import SolverConfig, gvns
    from .model import GeneratorConfig, generate_instance

    out = {}

    def vnd_ms(K, T, reps=3, variant=0):
        dev = _native.DeviceInstance.generate(GeneratorConfig(products=K, periods=T, seed=0))
        if variant:
            dev.set_variant(variant)
        sm, sr = dev.initial_solution()
        dev.vnd(sm, sr)
        best, st, tr = None, None, None
        for _ in range(reps):
            _, _, tr, st = dev.vnd(sm, sr)
            ms = st["kernel_ns"] / 1e6
            best = ms if best is None else min(best, ms)
        return dev, best, st, tr

    _, ms, st, _ = vnd_ms(1000, 52)
    out["c2_vnd"] = {"kernel_ms": ms, "cost": st["cost"], "bit_exact": st["cost"] == 4484593955,
                     "evals_reference": st["evals_reference"]}
    dev, ms, st, _ = vnd_ms(100000, 52, reps=3, variant=16)
    out["c3_int64"] = {"kernel_ms": ms, "cost": st["cost"],
                       "value_type_bytes": dev.info["value_bytes"],
                       "cost_type_bytes": dev.info["cost_bytes"],
                       "bit_exact": st["cost"] == 449100704810,
                       "reference_equiv_evals_per_s": st["evals_reference"] / (ms / 1e3)}
    del dev
    _, ms, st, tr = vnd_ms(10000, 520, reps=2)
    g4 = _golden("c4_full.json")
    out["c4_vnd"] = {"kernel_ms": ms, "cost": st["cost"], "sweeps": st["sweeps"],
                     "evals_reference": st["evals_reference"],
                     "reference_equiv_evals_per_s": st["evals_reference"] / (ms / 1e3),
                     "bit_exact": None if g4 is None else (
                         st["cost"] == g4["cost"] and tr.tolist() == g4["trace"]
                         and st["evals_reference"] == g4["evals"])}
    if roofline is not None:
        out["c4_vnd"]["roofline"] = roofline("c4", ms)

    inst2 = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    for name, W, R in (("c2_gvns", 2, 400), ("c2_gvns_20k", 2, 20000),
                       ("c5_gvns_1gpu_share", 128, 200), ("c5_gvns_all_1024", 1024, 40)):
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
    g5 = _golden("gvns_c5.json") or {}
    for name, W, R in (("W128_R4", 128, 4), ("W1024_R2", 1024, 2)):
        res = gvns(inst2, SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=W, seed=0,
                                       max_rounds=R))
        g = g5.get(name)
        out.setdefault("c5_parity", {})[name] = {
            "cost": res.cost, "bit_exact": None if g is None else (
                res.cost == g["cost"] and res.rounds == g["rounds"]
                and _plan_sha(res.plan.setup_m, res.plan.setup_r) == g["plan_sha"])}
    return out
