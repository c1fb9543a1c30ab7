"""Round-2 parity pins for the configs round 1 left unpinned.

Run in the build container only (the live reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/gen_pins_r02.py {c4,n2,int64,c5} ...

Instances come from the LIVE reference generator (``remlot.generate_instance``,
reference model.py:115-153) and start from its ``initial_solution``
(plan.py:140-167).  The descents are run by

* ``c4``, ``n2``, ``int64``: the C oracle (oracle/remlot_oracle.c, the
  lockstep restatement of vnd.py:253-289 over _kernels.py:46-344, itself
  pinned to the live reference by tests/test_oracle_golden.py).  A live
  numba run of full C4 is ~80 min on 8 threads; the oracle's is ~42 min.
* ``c5``: the live reference ``gvns`` itself (gvns.py:184-221) with the
  round cap of SolverConfig.max_rounds, W = 128 and 1,024 workers
  (Algorithm 2's W generalised).

Outputs (small JSON under tests/golden/):
  c4_full.json       K=10,000 T=520 seed 0: cost, start cost, 1,605-entry
                     trace, evals / moves / sweeps, plan sha256, per-product
                     final-cost sha256
  n2_weak.json       K=200,000 T=52 seed 0 (the N=2 weak-scaling instance of
                     bench.py: ranks 0/1 own products [0,1e5) and [1e5,2e5))
  int64_k10000.json  K=10,000 T=52 instances whose cost bound forces the
                     int64-cost path (int32 and int64 values)
  gvns_c5.json       K=1,000 T=52 gvns(seed 0): W=128 x 4 and W=1,024 x 2 rounds
  gvns_long.json     round-capped live gvns at horizons past the register
                     rows (T = 100, 300, 520: shared-memory rows in the
                     device shake / VND tasks) and with int64 costs
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import remlot  # noqa: E402  (the live reference)
from remlot import (GeneratorConfig, SolverConfig, generate_instance, gvns,  # noqa: E402
                    initial_solution)

assert "/root/reference" in os.path.dirname(remlot.__file__), remlot.__file__

from oracle import oracle as orc  # noqa: E402

THREADS = len(os.sched_getaffinity(0))


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def plan_sha(sm, sr):
    return sha(np.packbits(np.asarray(sm, bool)), np.packbits(np.asarray(sr, bool)))


def oracle_descent(cfg):
    inst = generate_instance(cfg)
    start = initial_solution(inst)
    t0 = time.time()
    sm, sr, cost, trace, st = orc.vnd(inst, start.setup_m, start.setup_r, 4, THREADS)
    wall = time.time() - t0
    final = orc.product_costs(inst, sm, sr)
    return dict(products=cfg.products, periods=cfg.periods, seed=cfg.seed,
                demand_max=cfg.demand_max,
                setup_cost_range=list(cfg.setup_cost_range),
                holding_cost_range=list(cfg.holding_cost_range),
                unit_cost_range=list(cfg.unit_cost_range),
                instance_sha=sha(inst.demand, inst.returns),
                start_plan_sha=plan_sha(start.setup_m, start.setup_r),
                start_cost=int(trace[0]), cost=int(cost), trace=[int(x) for x in trace],
                evals=st["evals"], moves=st["moves"], sweeps=st["sweeps"],
                plan_sha=plan_sha(sm, sr), product_costs_sha=sha(final),
                oracle_threads=THREADS, wall_s=round(wall, 1))


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, indent=1)
    print("wrote", name, flush=True)


def gen_c4():
    d = oracle_descent(GeneratorConfig(products=10000, periods=520, seed=0))
    print("C4", d["cost"], d["evals"], d["sweeps"], d["wall_s"], flush=True)
    dump("c4_full.json", d)


def gen_n2():
    d = oracle_descent(GeneratorConfig(products=200000, periods=52, seed=0))
    print("N2", d["cost"], d["evals"], d["sweeps"], d["wall_s"], flush=True)
    dump("n2_weak.json", d)


def gen_int64():
    out = {}
    # int32 values, costs beyond the int32 proof (T (k_M + k_R) alone > 2^30)
    out["v32_c64"] = oracle_descent(GeneratorConfig(
        products=10000, periods=52, seed=3, setup_cost_range=(50_000_000, 200_000_000)))
    # int64 values: sum D + sum R per product beyond 2^28
    out["v64_c64"] = oracle_descent(GeneratorConfig(
        products=10000, periods=52, seed=4, demand_max=20_000_000,
        setup_cost_range=(5_000_000_000, 20_000_000_000), holding_cost_range=(100, 500)))
    for k, d in out.items():
        print(k, d["cost"], d["evals"], d["sweeps"], d["wall_s"], flush=True)
    dump("int64_k10000.json", out)


def gen_c5():
    from remlot import _kernels
    _kernels.warm_up()
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    out = {}
    for W, R in ((128, 4), (1024, 2)):
        cfg = SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=W, seed=0,
                           max_rounds=R, vnd_mode="serial", parallelism=1)
        t0 = time.time()
        res = gvns(inst, cfg)
        out[f"W{W}_R{R}"] = dict(cost=int(res.cost), rounds=res.rounds,
                                 shake_calls=res.shake_calls,
                                 plan_sha=plan_sha(res.plan.setup_m, res.plan.setup_r),
                                 wall_s=round(time.time() - t0, 1))
        print("C5", W, R, res.cost, time.time() - t0, flush=True)
        dump("gvns_c5.json", out)


def gen_long():
    from remlot import _kernels
    _kernels.warm_up()
    cases = {
        "K40_T100_W2_R30": (GeneratorConfig(products=40, periods=100, seed=11), 2, 30),
        "K16_T300_W3_R12": (GeneratorConfig(products=16, periods=300, seed=12), 3, 12),
        "K12_T520_W2_R8": (GeneratorConfig(products=12, periods=520, seed=13), 2, 8),
        "K20_T100_c64_W2_R10": (GeneratorConfig(products=20, periods=100, seed=14,
                                                setup_cost_range=(50_000_000, 200_000_000)),
                                2, 10),
    }
    out = {}
    for name, (gc, W, R) in cases.items():
        inst = generate_instance(gc)
        cfg = SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=W, seed=5,
                           max_rounds=R, vnd_mode="serial", parallelism=1)
        t0 = time.time()
        res = gvns(inst, cfg)
        out[name] = dict(products=gc.products, periods=gc.periods, seed=gc.seed,
                         setup_cost_range=list(gc.setup_cost_range), workers=W, rounds=R,
                         cost=int(res.cost), rounds_done=res.rounds,
                         shake_calls=res.shake_calls,
                         plan_sha=plan_sha(res.plan.setup_m, res.plan.setup_r),
                         instance_sha=sha(inst.demand, inst.returns),
                         wall_s=round(time.time() - t0, 1))
        print("long", name, res.cost, res.rounds, res.shake_calls, time.time() - t0, flush=True)
    dump("gvns_long.json", out)


if __name__ == "__main__":
    jobs = dict(c4=gen_c4, n2=gen_n2, int64=gen_int64, c5=gen_c5, long=gen_long)
    for a in sys.argv[1:]:
        jobs[a]()
