#!/usr/bin/env python
"""Benchmark of the VND hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3|c2|c4] [--scaling weak|strong]

Workload (BASELINE.json configs[2], the config the metric "neighbor
evals/sec & VND time-to-local-opt at 1/2/4/8 B200" is quoted on): the
seed-0 synthetic instance K=100,000 products x T=52 periods, VND (N1..N4) to
the local optimum from the lot-for-lot start.  A step is one full descent.

Multi-GPU: ``--gpus N`` with no WORLD_SIZE in the environment re-launches
itself under torch.distributed.run with N ranks (one per GPU); under
torchrun the world size must equal --gpus.  Products are sharded in
contiguous blocks with no data-path collective (one all-reduce of the
totals).  Default --scaling weak: the job instance is the seed-0 generator
instance with K = 100,000 x N products and every rank descends its own
100,000 (N=1 is exactly BASELINE config 3); the line also carries
``strong``: the fixed K=100,000 of config 3 sharded over the N ranks.

value   = reference-equivalent neighbor evaluations (the reference's lockstep
          count) per second, whole job, inputs resident.
e2e     = same metric through the C ABI with host (pinned) buffers: every
          step re-uploads the instance and the start plan and reads back the
          final plan, trace and stats.
roofline = the VND kernel against the SM instruction-issue ceiling (warp
          instructions of one launch, from the committed ncu capture of this
          build, / the live kernel time, vs SMs x 4 schedulers x clock);
          the 8T-ops figure is kept as ``formulation_relative``.
--impl reference = the CPU reference path (oracle/, a C restatement of the
          reference's numba kernels run product-parallel on every host core)
          on the same full instance.
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c3": dict(products=100_000, periods=52, name="K=100000 T=52 seed0 VND-to-local-opt"),
    "c2": dict(products=1_000, periods=52, name="K=1000 T=52 seed0 VND-to-local-opt"),
    "c4": dict(products=10_000, periods=520, name="K=10000 T=520 seed0 VND-to-local-opt"),
}
L2_BYTES = 126 * 1024 * 1024
METRIC = "neighbor evals/sec (reference-equivalent) & VND time-to-local-opt"


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sms, maxes, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sms.append(float(parts[0]))
                maxes.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(name)
        if not sms:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sms)), "sm_max_mhz": max(maxes),
                "reasons": sorted(reasons), "samples": len(sms)}


def cpu_reference(inst, sample_products, steps, warmup, threads):
    """Time the CPU reference path (oracle port) on the first products."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    oracle.lib()
    sub = inst.slice(0, sample_products)
    oi = oracle.OracleInstance(sub)
    sm, sr = oracle.initial_solution(oi)
    times, stats = [], None
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        _, _, cost, _, stats = oracle.vnd(oi, sm, sr, 4, threads)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    t = float(np.mean(times))
    return dict(value=stats["evals"] / t, evals=stats["evals"], seconds_per_step=t, cost=cost,
                sweeps=stats["sweeps"])


def cpu_gvns_reference(threads, workers=2, budget_s=10.0):
    """GVNS rounds/s of the CPU reference path at C2 (K=1000, T=52, W=2,
    k_max=5, seed 0): the port of gvns.py:147-221 (oracle/gvns_oracle.py:
    numpy-exact shake + the C oracle's VND), the W workers of a round on W
    host threads like the reference's ThreadPoolExecutor; as many rounds as
    fit in ~budget_s."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from concurrent.futures import ThreadPoolExecutor

    import gvns_oracle
    import numpy_rng
    import oracle
    from paper_1704_05132_b200.model import GeneratorConfig, generate_instance
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    oi = oracle.OracleInstance(inst)
    init = oracle.initial_solution(oi)
    inc = (init[0].copy(), init[1].copy())
    inc_cost = oracle.evaluate(oi, *inc)
    k, k_max, rounds = 1, 5, 0

    def work(r, w, plan, k):
        rng = numpy_rng.Philox.from_entropy((0, r, w))
        m, s = gvns_oracle.shake(oi, plan[0], plan[1], init, k, rng)
        m, s, cost, _, _ = oracle.vnd(oi, m, s, 4)
        return cost, w, m, s

    t0 = time.perf_counter()
    with ThreadPoolExecutor(workers) as pool:
        while time.perf_counter() - t0 < budget_s:
            res = list(pool.map(lambda w: work(rounds, w, inc, k), range(workers)))
            cost, _, m, s = min(res, key=lambda x: (x[0], x[1]))
            rounds += 1
            improved = cost < inc_cost
            if improved:
                inc, inc_cost = (m, s), cost
            k = 1 if improved or k >= k_max else k + 1
    dt = time.perf_counter() - t0
    return {"value": rounds / dt, "unit": "rounds/s", "cores": min(workers, threads),
            "kind": "port", "rounds": rounds, "best_cost": int(inc_cost),
            "sample": f"{rounds} GVNS rounds from the lot-for-lot start (W={workers}, "
                      f"k_max={k_max}, seed 0) in {dt:.1f} s; shake in Python (numpy-exact "
                      "Philox restatement) + C oracle VND, one host thread per worker"}


def sharded_c5(torch, dist, coll, rank, rounds=40):
    """BASELINE config 5 on the job's ranks: sharded_gvns with W=1,024 over
    K=1000 T=52 (seed 0): bit-exactness against the W1024_R2 golden, then
    rounds/s of a `rounds`-round run (wall clock around the call, device
    synchronised, max over ranks)."""
    from paper_1704_05132_b200 import GeneratorConfig, SolverConfig, generate_instance
    from paper_1704_05132_b200.sharded import sharded_gvns
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    out = {"workers": 1024, "products": 1000, "periods": 52}
    try:
        with open(os.path.join(ROOT, "tests", "golden", "gvns_c5.json")) as f:
            g = json.load(f)["W1024_R2"]
    except (OSError, KeyError, ValueError):
        g = None
    res = sharded_gvns(inst, SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=1024,
                                          seed=0, max_rounds=2))
    if g is not None:
        import hashlib
        h = hashlib.sha256()
        h.update(np.packbits(res.plan.setup_m).tobytes())
        h.update(np.packbits(res.plan.setup_r).tobytes())
        out["bit_exact_W1024_R2"] = res.cost == g["cost"] and h.hexdigest() == g["plan_sha"]
    cfg = SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=1024, seed=0, max_rounds=rounds)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = sharded_gvns(inst, cfg)
    torch.cuda.synchronize()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=coll)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    sec = float(dt[0])
    out.update(rounds=res.rounds, seconds=sec, rounds_per_s=res.rounds / sec,
               shakes_per_s=res.shake_calls / sec, best_cost=res.cost,
               timing="wall clock around sharded_gvns, device-synchronised, max over ranks")
    return out


def hbm_bytes(wl):
    """Algorithmic HBM bytes of one VND launch per GPU:
    int32 D, R rows + six int64 cost vectors + plan in/out bytes."""
    K, T = wl["products"], wl["periods"]
    return K * (8 * T + 48) + K * 2 * T * 2


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 7700.0   # B200_PROFILING.md fallback


def ncu_summary(workload):
    """Issue-slot / pipe utilisation of k_vnd from the committed ncu --set
    full capture of this workload (profiles/k_vnd_<workload>_ncu.json)."""
    path = os.path.join(ROOT, "profiles", f"k_vnd_{workload}_ncu.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def traffic_bytes(workload):
    """dram__bytes_read.sum + dram__bytes_write.sum of one k_vnd launch on
    this workload from the committed ncu --set full capture (profiles/), or
    None when no capture of the current round exists."""
    path = os.path.join(ROOT, "profiles", f"k_vnd_{workload}_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)["bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def relaunch(n):
    """Start n ranks of this command under torch.distributed.run (one per
    GPU, rendezvous on 127.0.0.1) and return its exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")   # the communicator shows in the logs
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def issue_roofline(workload, kernel_ms, clocks, sms):
    """The VND kernel against the SM instruction-issue ceiling: warp
    instructions per launch (deterministic work; from the committed ncu
    capture of this build, profiles/k_vnd_<wl>_ncu.json) / the live kernel
    time, against SMs x 4 schedulers x the SM clock under load."""
    ncu = ncu_summary(workload)
    if not ncu or not ncu.get("warp_inst"):
        return None
    mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    peak = sms * 4 * mhz * 1e6
    achieved = ncu["warp_inst"] / (kernel_ms / 1e3)
    lanes = ncu.get("threads_pred_on_per_inst") or ncu.get("threads_per_inst")
    return {"bound": "sm_issue", "kernel": "k_vnd", "achieved": achieved / 1e9,
            "peak": peak / 1e9, "unit": "Gwarp-inst/s", "frac": achieved / peak,
            "peak_source": f"{sms} SMs x 4 schedulers x {mhz:.0f} MHz (SM clock under load)",
            "warp_inst_per_launch": ncu["warp_inst"], "kernel_ms": kernel_ms,
            "threads_per_inst_frac": (lanes / 32.0) if lanes else None,
            "threads_note": "not-predicated threads per issued instruction / 32 (ncu); since "
                            "round 2 the walk step is issued unconditionally, so this counts "
                            "idle lanes issuing the discarded step -- the walk's useful-lane "
                            "share is ~0.46 at C3 (tools/walk_stats.py, DESIGN.md 5)",
            "traffic": traffic_bytes(workload), "ncu": ncu}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="reference arm: products of the workload instance per timed step "
                         "(0 = all of it, the same config as ours)")
    ap.add_argument("--scaling", default="weak", choices=("weak", "strong"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the secondary configs (C2 GVNS, C4, C5 share)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args.gpus)
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    wl = WORKLOADS[args.workload]
    from paper_1704_05132_b200.model import GeneratorConfig, generate_instance

    threads = len(os.sched_getaffinity(0))
    if args.impl == "reference":
        if rank != 0:
            return 0
        inst = generate_instance(GeneratorConfig(products=wl["products"], periods=wl["periods"],
                                                 seed=0))
        sample = wl["products"] if args.cpu_sample <= 0 else min(args.cpu_sample, wl["products"])
        # the C port has nothing to warm up (no JIT): warm-up steps descend
        # a 2,000-product prefix, every timed step the whole workload
        cpu_reference(inst, min(2000, sample), 0, args.warmup, threads)
        r = cpu_reference(inst, sample, args.steps, 0, threads)
        full = sample == wl["products"]
        line = {
            "impl": "reference", "metric": METRIC,
            "value": r["value"], "unit": "evals/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["seconds_per_step"] * 1e3,
            "time_to_local_opt_ms": r["seconds_per_step"] * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "int64", "data": "synthetic (reference generator, seed 0)",
            "config": {"workload": wl["name"], "products": wl["products"],
                       "periods": wl["periods"], "k_max": 4, "parallelism": "cpu-threads"},
            "same_config": full,
            "cpu_baseline": {"value": r["value"], "unit": "evals/s", "cores": threads,
                             "kind": "port",
                             "sample": (f"the whole workload instance ({sample} products)"
                                        if full else f"first {sample} products of the workload "
                                        "instance") + ", lockstep VND to local optimum from "
                                        "the lot-for-lot start (oracle/remlot_oracle.c, pthreads "
                                        "product-parallel); warm-up steps on a 2,000-product "
                                        "prefix"},
            "e2e": {"value": r["value"], "unit": "evals/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "evals_reference_per_step": r["evals"], "final_cost": r["cost"],
        }
        if full and args.workload == "c3":
            line["parity"] = {"final_cost": r["cost"], "reference_final_cost": 449100704810,
                              "bit_exact": r["cost"] == 449100704810,
                              "evals_reference_golden": r["evals"] == 878715402}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist
    from paper_1704_05132_b200 import _native
    from paper_1704_05132_b200 import devbench, sharded

    # RL_BENCH_BACKEND=gloo runs the multi-rank plumbing with several ranks
    # on one GPU (test only: NCCL refuses two ranks per device); collectives
    # then go through host tensors.
    backend = os.environ.get("RL_BENCH_BACKEND", "nccl")
    dev_idx = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev_idx)
    coll = "cuda" if backend == "nccl" else "cpu"
    if world > 1:
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")   # the driver's rank check reads it
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
        else:
            dist.init_process_group(backend)
    K0, T = wl["products"], wl["periods"]
    stream = torch.cuda.Stream()   # a real stream: events and kernels share it
    torch.cuda.set_stream(stream)
    sptr = ctypes.c_void_p(stream.cuda_stream)
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device="cuda")
    lib = _native.load()

    def measure(K, steps, warmup, sample_clocks):
        """Time `steps` descents of this rank's shard of the seed-0 K-product
        instance: device events per step on the launching stream (L2 flushed
        between steps), max over ranks; totals combined like the reference's
        lockstep loop (sharded.combine)."""
        lo, hi = sharded.shard_bounds(K, rank, world)
        # each rank draws only its shard of the seed-0 instance on its device
        # (rl_generate_instance: bit-identical to generate_instance, tested)
        dev = _native.DeviceInstance.generate(GeneratorConfig(products=K, periods=T, seed=0),
                                              lo, hi)
        plan = torch.empty((4, hi - lo, T), dtype=torch.uint8, device="cuda")
        pp = [ctypes.c_void_p(plan[i].data_ptr()) for i in range(4)]
        _native.check(lib.rl_initial_solution_device(dev.h, pp[0], pp[1], sptr),
                      "rl_initial_solution_device")

        def step():
            _native.check(lib.rl_vnd_device(dev.h, 4, *pp, sptr), "rl_vnd_device")

        def collect():
            tr = np.empty(1 << 16, np.int64)
            nt = np.zeros(1, np.int64)
            st = np.zeros(9, np.int64)
            _native.check(lib.rl_vnd_collect(dev.h, _native.ptr(tr), len(tr), _native.ptr(nt),
                                             _native.ptr(st)), "rl_vnd_collect")
            return tr[:nt[0]].tolist(), dict(evals=int(st[3]), evals_reference=int(st[4]),
                                             moves=int(st[5]), ntot_sum=int(st[8]), k_max=4,
                                             kernel_ns=int(st[7]))

        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        collect()
        sampler = ClockSampler(dev_idx) if sample_clocks else None
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if sampler:
            sampler.start()
        launches0 = dev.launches
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        kernel_ms = []
        for e0, e1 in evs:
            flush.zero_()
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            kernel_ms.append(collect()[1]["kernel_ns"] / 1e6)
        torch.cuda.synchronize()
        launches = dev.launches - launches0
        if world > 1:
            dist.barrier()
        clocks = sampler.stop() if sampler else None
        my_ms = float(np.sum([e0.elapsed_time(e1) for e0, e1 in evs]))
        trace, stats = collect()
        tmax = torch.tensor([my_ms, float(np.mean(kernel_ms))], dtype=torch.float64,
                            device=coll)
        if world > 1:
            g_trace, totals = sharded.combine(trace, stats, device=coll)
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        else:
            g_trace, totals = trace, dict(evals_reference=stats["evals_reference"],
                                          evals=stats["evals"], cost=trace[-1],
                                          moves=stats["moves"])
        total_ms, vnd_kernel_ms = tmax.tolist()
        return dict(dev=dev, K=K, lo=lo, hi=hi, total_ms=total_ms, kernel_ms=vnd_kernel_ms,
                    ms_per_step=total_ms / steps, launches=launches, clocks=clocks,
                    trace=g_trace, totals=totals,
                    value=totals["evals_reference"] * steps / (total_ms / 1e3))

    K = K0 * world if args.scaling == "weak" else K0
    m = measure(K, args.steps, args.warmup, True)
    dev = m["dev"]
    totals = m["totals"]
    ref_evals, done_evals = totals["evals_reference"], totals["evals"]
    final_cost, moves = totals["cost"], totals["moves"]
    ms_per_step = m["ms_per_step"]
    clocks = m["clocks"]
    # ---- e2e through the C ABI with pinned host buffers
    shard = dev.download()
    e2e_ms, h2d, d2h = devbench.e2e_steps(torch, _native, dev, shard, args.steps, world, dist,
                                          coll)
    # ---- the other scaling mode at N > 1 (config 3 is the fixed K=100,000)
    other = None
    if world > 1:
        other = measure(K0 if args.scaling == "weak" else K0 * world, args.steps, args.warmup,
                        False)

    # ---- BASELINE config 5 across the ranks: 1,024 replicas of K=1000 T=52
    # (sharded.sharded_gvns: worker blocks per rank, speculative batches, one
    # all-gather per batch), parity against the live reference's round-capped
    # golden and rounds/s over a longer run
    c5 = None
    if world > 1 and not args.no_extra:
        c5 = sharded_c5(torch, dist, coll, rank)

    line = None
    if rank == 0:
        value = m["value"]
        alg_ops = done_evals * 8 * T / world   # 8T int ops per evaluation
        achieved = alg_ops / (m["kernel_ms"] / 1e3)
        peak_ops = devbench.int32_peak_ops()
        roof = issue_roofline(args.workload, m["kernel_ms"], clocks, dev.info["sms"]) \
            if world == 1 and K == K0 else None
        if roof is None:   # per-rank work differs from the captured launch
            roof = {"bound": "sm_issue", "kernel": "k_vnd", "achieved": None, "peak": None,
                    "unit": "Gwarp-inst/s", "frac": None, "kernel_ms": m["kernel_ms"],
                    "traffic": traffic_bytes(args.workload),
                    "note": "ncu capture is of the N=1 launch"}
        roof["formulation_relative"] = {
            "achieved": achieved / 1e9, "peak": peak_ops / 1e9, "unit": "Gop/s",
            "frac": achieved / peak_ops,
            "definition": "8*T int ops per performed neighbor evaluation (the reference's "
                          "per-period recurrence, SURVEY.md 8(d)) / kernel time, vs the "
                          "in-bench INT32 IMAD+LOP3 microbenchmark; the delta walk executes "
                          "far fewer ops, so this measures the formulation, not the kernel"}
        roof["hbm"] = {"achieved": hbm_bytes(wl) * world / (m["kernel_ms"] / 1e3) / 1e9,
                       "peak": hbm_peak(), "unit": "GB/s",
                       "note": "algorithmic bytes (instance + plans once) per launch / "
                               "kernel time: not the binding resource"}
        line = {
            "metric": METRIC,
            "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step,
            "time_to_local_opt_ms": ms_per_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "int32" if dev.info["cost_bytes"] == 4 else "int64",
            "data": "synthetic (reference generator model.py:115-153, seed 0)",
            "config": {"workload": wl["name"] if world == 1 else
                       f"K={K} T={T} seed0 VND-to-local-opt ({K // world} products per GPU)",
                       "products": K, "periods": T, "k_max": 4,
                       "parallelism": f"product-shard x{world}",
                       "l2": "flushed between steps (256 MiB write)",
                       "cost_type_bytes": dev.info["cost_bytes"],
                       "value_type_bytes": dev.info["value_bytes"]},
            "evals_reference_per_step": ref_evals, "evals_performed_per_step": done_evals,
            "performed_evals_per_s": done_evals * args.steps / (m["total_ms"] / 1e3),
            "final_cost": final_cost, "moves_per_step": moves,
            "gpu_launches": int(m["launches"]) * world,
            "clocks": clocks,
            "e2e": {"value": ref_evals * args.steps / (e2e_ms / 1e3), "unit": "evals/s",
                    "ms_per_step": e2e_ms / args.steps, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "roofline": roof,
        }
        if c5 is not None:
            line["c5_sharded"] = c5
        if other is not None:
            line["strong" if args.scaling == "weak" else "weak"] = {
                "products": other["K"], "value": other["value"], "unit": "evals/s",
                "ms_per_step": other["ms_per_step"],
                "time_to_local_opt_ms": other["ms_per_step"],
                "final_cost": other["totals"]["cost"],
                "evals_reference_per_step": other["totals"]["evals_reference"],
                "bit_exact": (other["totals"]["cost"] == 449100704810
                              if other["K"] == K0 else None)}
        if world == 1 and not args.no_cpu_baseline:
            inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=0))
            # bounded sample sized for ~10-20 s of CPU work on this host
            probe = cpu_reference(inst, min(1000, K), 1, 0, threads)
            per_product = probe["seconds_per_step"] / min(1000, K)
            sample = int(min(K, max(1000, 12.0 / max(per_product, 1e-9))))
            r = cpu_reference(inst, sample, 1, 0, threads)
            # and one core (serial and product-parallel)
            s1 = max(100, min(K, int(sample * 3.0 / max(r["seconds_per_step"] * threads, 1e-9))))
            r1 = cpu_reference(inst, s1, 1, 0, 1)
            line["cpu_baseline"] = {
                "value": r["value"], "unit": "evals/s", "cores": threads, "kind": "port",
                "sample": f"first {sample} products, lockstep VND to local optimum "
                          f"({r['seconds_per_step']:.2f} s)",
                "serial": {"value": r1["value"], "cores": 1,
                           "sample": f"first {s1} products ({r1['seconds_per_step']:.2f} s)"}}
        if world == 1 and not args.no_extra:
            line["other_configs"] = oc = devbench.other_configs(
                torch, clocks, roofline=lambda w, ms: issue_roofline(w, ms, clocks,
                                                                     dev.info["sms"]))
            if not args.no_cpu_baseline:
                # C4's CPU reference rate on a bounded sample (the full run
                # is ~40 min on 8 threads of the port)
                inst4 = generate_instance(GeneratorConfig(products=10000, periods=520, seed=0))
                n4 = 4 * threads
                r4 = cpu_reference(inst4, n4, 1, 0, threads)
                oc["c4_vnd"]["cpu_baseline"] = {
                    "value": r4["value"], "unit": "evals/s", "cores": threads, "kind": "port",
                    "sample": f"first {n4} products, VND to local optimum "
                              f"({r4['seconds_per_step']:.2f} s)"}
                oc["c2_gvns"]["cpu_baseline"] = cpu_gvns_reference(threads)
        golden = {100_000: (449100704810, 878715402)}
        try:
            with open(os.path.join(ROOT, "tests", "golden", "n2_weak.json")) as f:
                g2 = json.load(f)
            golden[g2["products"]] = (g2["cost"], g2["evals"])
        except (OSError, ValueError, KeyError):
            pass
        if args.workload == "c3" and K in golden:
            line["parity"] = {"final_cost": final_cost, "reference_final_cost": golden[K][0],
                              "bit_exact": final_cost == golden[K][0],
                              "evals_reference_golden": ref_evals == golden[K][1]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
