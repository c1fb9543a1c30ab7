"""Generate the golden fixtures under tests/golden/ from the LIVE reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/gen_golden.py [--big]

Everything here calls the reference package ``remlot`` through its public
API or its numba kernels (``remlot._kernels``); nothing from this repo is
imported, so the fixtures are an independent pin for the oracle (oracle/)
and for the CUDA path.  ``--big`` adds the K=100,000 x T=52 run (~90 s on
8 cores) and the T=520 product sample.

Fixture files (all small; plans of large runs are stored as sha256 of
np.packbits(setup_m) || np.packbits(setup_r)):
  instances.json     sha256 of generated instance arrays per GeneratorConfig
  small_cases.npz    random small instances/plans: row costs, list_moves,
                     scan_products outputs per nbh, vnd (plan, cost, trace)
  c1_trajectory.npz  K=10 T=52 seed 0: scan outputs of every lockstep pass
  k1000.npz          K=1000 T=52 seed 0: vnd final plan/cost/trace/stats
  big.json           K=100000 T=52 and T=520 sample summaries (--big)
  rng.npz            numpy Philox/SeedSequence/choice/shuffle streams
  gvns_small.npz     shake / worker_round / gvns(max_rounds) results
  gvns_k1000.json    K=1000 T=52 gvns(seed=0): W=2 x 20 and x 150 rounds, W=16 x 4
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

import remlot
from remlot import (GeneratorConfig, Instance, SetupPlan, SolverConfig,
                    generate_instance, gvns, initial_solution, shake, vnd,
                    worker_round)
from remlot import _kernels
from remlot.gvns import _worker_rng
from remlot.vnd import _move_buffers, _run_scan, _scan_outputs

HERE = os.path.dirname(os.path.abspath(__file__))
assert "/root/reference" in os.path.dirname(remlot.__file__), remlot.__file__


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def plan_sha(sm, sr):
    return sha(np.packbits(np.asarray(sm, bool)), np.packbits(np.asarray(sr, bool)))


def inst_arrays(inst):
    return dict(demand=inst.demand, returns=inst.returns,
                setup_cost_m=inst.setup_cost_m, setup_cost_r=inst.setup_cost_r,
                holding_cost_m=inst.holding_cost_m, holding_cost_r=inst.holding_cost_r,
                unit_cost_m=inst.unit_cost_m, unit_cost_r=inst.unit_cost_r)


def cost_args(inst):
    return (inst.setup_cost_m, inst.setup_cost_r, inst.holding_cost_m,
            inst.holding_cost_r, inst.unit_cost_m, inst.unit_cost_r)


def row_costs(inst, sm, sr):
    out = np.empty(inst.products, np.int64)
    _kernels.product_costs(0, inst.products, sm, sr, inst.demand, inst.returns,
                           *cost_args(inst), out)
    return out


def scan(inst, sm, sr, nbh):
    out = _scan_outputs(inst.products)
    _run_scan(inst, sm, sr, nbh, "serial", 1, out)
    return out


def list_moves_all(sm, sr, nbh):
    """Per product move lists, padded to 2T (canonical reference order)."""
    K, T = sm.shape
    n = np.zeros(K, np.int64)
    bufs = [np.zeros((K, 2 * T), np.int64), np.zeros((K, 2 * T), bool),
            np.zeros((K, 2 * T), bool), np.full((K, 2 * T), -1, np.int64),
            np.zeros((K, 2 * T), bool), np.zeros((K, 2 * T), bool)]
    for k in range(K):
        mp0, mm0, mr0, mp1, mm1, mr1 = _move_buffers(T)
        c = _kernels.list_moves(nbh, sm[k], sr[k], mp0, mm0, mr0, mp1, mm1, mr1)
        n[k] = c
        for dst, src in zip(bufs, (mp0, mm0, mr0, mp1, mm1, mr1)):
            dst[k, :c] = src[:c]
        # single-period moves leave mm1/mr1 unwritten in the reference
        single = bufs[3][k, :c] < 0
        bufs[4][k, :c][single] = False
        bufs[5][k, :c][single] = False
    return n, bufs


def lockstep_vnd(inst, plan, k_max=4, record=False):
    """The reference vnd() loop (vnd.py:253-289) replayed through the
    reference kernels, also counting candidate evaluations (list_moves n for
    feasible products, _kernels.py:284-294) and optionally recording every
    pass's scan outputs."""
    sm = plan.setup_m.copy()
    sr = plan.setup_r.copy()
    K = inst.products
    cost = remlot.evaluate(inst, plan)
    trace = [cost]
    evals = 0
    moves = 0
    sweeps = 0
    rec = []
    bufs = _move_buffers(inst.periods)
    while True:
        sweeps += 1
        improvement = False
        for nbh in range(1, k_max + 1):
            feas = row_costs(inst, sm, sr) != remlot.INFEASIBLE
            for k in np.flatnonzero(feas):
                evals += _kernels.list_moves(nbh, sm[k], sr[k], *bufs)
            out = scan(inst, sm, sr, nbh)
            if record:
                rec.append(tuple(np.array(a) for a in out))
            moves += int((out[0] > 0).sum())
            diff = int(_kernels.apply_scan(0, K, *out, sm, sr))
            if diff > 0:
                cost -= diff
                improvement = True
            trace.append(cost)
        if not improvement:
            break
    ref_plan, ref_cost = vnd(inst, plan, k_max, mode="product-parallel",
                             parallelism=8)
    assert ref_cost == cost and np.array_equal(ref_plan.setup_m, sm)
    return sm, sr, cost, np.array(trace, np.int64), evals, moves, sweeps, rec


def random_instance(seed, products=3, periods=6, demand_max=9, return_ratio=0.6,
                    **kw):
    return generate_instance(GeneratorConfig(
        products=products, periods=periods, demand_max=demand_max,
        return_ratio=return_ratio, seed=seed, **kw))


def gen_instances():
    cfgs = [dict(products=10, periods=52, seed=0),
            dict(products=1000, periods=52, seed=0),
            dict(products=300, periods=52, seed=77),
            dict(products=100000, periods=52, seed=0),
            dict(products=10000, periods=520, seed=0),
            dict(products=3, periods=6, demand_max=9, return_ratio=0.6, seed=5),
            dict(products=130, periods=8, demand_max=9, return_ratio=0.6, seed=4000),
            dict(products=2, periods=5, demand_max=9, return_ratio=0.5,
                 setup_cost_range=(2000, 8000), holding_cost_range=(100, 500),
                 seed=1000),
            dict(products=4, periods=9, demand_max=0, seed=3),
            dict(products=5, periods=7, demand_max=50, return_ratio=1.0,
                 unit_cost_range=(5, 90), seed=2**40 + 7),
            dict(products=50, periods=52, seed=2003)]
    out = []
    for cfg in cfgs:
        inst = generate_instance(GeneratorConfig(**cfg))
        arrs = inst_arrays(inst)
        out.append(dict(config={k: (list(v) if isinstance(v, tuple) else v)
                                for k, v in cfg.items()},
                        sha256={k: sha(v) for k, v in arrs.items()},
                        demand_sum=int(inst.demand.sum()),
                        returns_sum=int(inst.returns.sum())))
    with open(os.path.join(HERE, "instances.json"), "w") as f:
        json.dump(out, f, indent=1)


def gen_small_cases():
    rng = np.random.default_rng(20261018)
    data = {}
    cases = []
    specs = []
    for seed in range(40):
        K = int(rng.integers(1, 8))
        T = int(rng.integers(1, 13))
        specs.append((seed, K, T, float(rng.uniform(0.0, 1.0)),
                      int(rng.integers(0, 30))))
    # a few wider horizons exercising multi-word bit masks on device
    specs += [(100, 3, 64, 0.5, 40), (101, 2, 65, 0.7, 60), (102, 2, 97, 0.4, 100),
              (103, 2, 130, 0.5, 100), (104, 1, 200, 0.9, 9)]
    for idx, (seed, K, T, ratio, dmax) in enumerate(specs):
        inst = random_instance(seed, products=K, periods=T, demand_max=dmax,
                               return_ratio=ratio,
                               setup_cost_range=(100, 5000) if T < 20 else (50_000, 200_000))
        plans = [initial_solution(inst),
                 SetupPlan(rng.random((K, T)) < 0.5, rng.random((K, T)) < 0.5),
                 SetupPlan(np.ones((K, T), bool), rng.random((K, T)) < 0.4),
                 SetupPlan.all_false(K, T)]
        for pi, plan in enumerate(plans):
            p = f"c{idx}_{pi}_"
            if pi == 0:
                for k, v in inst_arrays(inst).items():
                    data[f"c{idx}_{k}"] = v
            data[p + "sm"] = plan.setup_m
            data[p + "sr"] = plan.setup_r
            data[p + "cost"] = row_costs(inst, plan.setup_m, plan.setup_r)
            for nbh in (1, 2, 3, 4):
                n, bufs = list_moves_all(plan.setup_m, plan.setup_r, nbh)
                data[p + f"lm{nbh}_n"] = n
                for name, b in zip(("mp0", "mm0", "mr0", "mp1", "mm1", "mr1"), bufs):
                    data[p + f"lm{nbh}_{name}"] = b
                out = scan(inst, plan.setup_m, plan.setup_r, nbh)
                for name, a in zip(("dec", "p0", "m0", "r0", "p1", "m1", "r1"), out):
                    a = np.array(a)
                    if name in ("m0", "r0"):
                        a = np.where(out[0] > 0, a, False)
                    if name in ("m1", "r1"):
                        a = np.where((out[0] > 0) & (out[4] >= 0), a, False)
                    data[p + f"scan{nbh}_{name}"] = a
            for k_max in (1, 4):
                trace = []
                vp, vc = vnd(inst, plan, k_max, trace=trace)
                data[p + f"vnd{k_max}_sm"] = vp.setup_m
                data[p + f"vnd{k_max}_sr"] = vp.setup_r
                data[p + f"vnd{k_max}_cost"] = np.int64(vc)
                data[p + f"vnd{k_max}_trace"] = np.array(trace, np.int64)
        cases.append((idx, K, T))
    data["cases"] = np.array(cases, np.int64)
    data["n_plans"] = np.int64(4)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **data)


def gen_c1():
    inst = generate_instance(GeneratorConfig(products=10, periods=52, seed=0))
    start = initial_solution(inst)
    sm, sr, cost, trace, evals, moves, sweeps, rec = lockstep_vnd(inst, start, record=True)
    data = dict(start_sm=start.setup_m, start_sr=start.setup_r, final_sm=sm,
                final_sr=sr, cost=np.int64(cost), trace=trace,
                evals=np.int64(evals), moves=np.int64(moves),
                sweeps=np.int64(sweeps))
    for name, i in zip(("dec", "p0", "m0", "r0", "p1", "m1", "r1"), range(7)):
        stack = np.stack([r[i] for r in rec])
        if name in ("m0", "r0"):
            stack = np.where(np.stack([r[0] for r in rec]) > 0, stack, False)
        if name in ("m1", "r1"):
            stack = np.where((np.stack([r[0] for r in rec]) > 0)
                             & (np.stack([r[4] for r in rec]) >= 0), stack, False)
        data["pass_" + name] = stack
    np.savez_compressed(os.path.join(HERE, "c1_trajectory.npz"), **data)
    print("C1", cost, sweeps, moves, evals, len(trace))


def gen_k1000():
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    start = initial_solution(inst)
    t0 = time.time()
    sm, sr, cost, trace, evals, moves, sweeps, _ = lockstep_vnd(inst, start)
    np.savez_compressed(os.path.join(HERE, "k1000.npz"),
                        start_sm=np.packbits(start.setup_m, axis=1),
                        start_sr=np.packbits(start.setup_r, axis=1),
                        final_sm=np.packbits(sm, axis=1), final_sr=np.packbits(sr, axis=1),
                        start_cost=np.int64(trace[0]), cost=np.int64(cost), trace=trace,
                        evals=np.int64(evals), moves=np.int64(moves),
                        sweeps=np.int64(sweeps))
    print("K1000", cost, sweeps, moves, evals, f"{time.time() - t0:.1f}s")


def gen_big():
    out = {}
    inst = generate_instance(GeneratorConfig(products=100000, periods=52, seed=0))
    start = initial_solution(inst)
    t0 = time.time()
    trace = []
    plan, cost = vnd(inst, start, mode="product-parallel", parallelism=8, trace=trace)
    out["k100000_t52"] = dict(start_cost=int(trace[0]), cost=int(cost),
                              sweeps=(len(trace) - 1) // 4, trace=[int(x) for x in trace],
                              start_plan_sha=plan_sha(start.setup_m, start.setup_r),
                              plan_sha=plan_sha(plan.setup_m, plan.setup_r),
                              wall_s=time.time() - t0)
    print("K100000", cost, time.time() - t0)
    # T=520: per-product VND is exact by decomposition, so a product subset
    # of the K=10000 instance pins the long-horizon path.
    inst = generate_instance(GeneratorConfig(products=10000, periods=520, seed=0))
    sub = [0, 1, 2, 3, 4, 5, 6, 7, 4999, 9999]
    sl = Instance(len(sub), 520, inst.demand[sub], inst.returns[sub],
                  inst.setup_cost_m[sub], inst.setup_cost_r[sub],
                  inst.holding_cost_m[sub], inst.holding_cost_r[sub],
                  inst.unit_cost_m[sub], inst.unit_cost_r[sub])
    start = initial_solution(sl)
    t0 = time.time()
    trace = []
    plan, cost = vnd(sl, start, mode="product-parallel", parallelism=8, trace=trace)
    out["k10000_t520_sample"] = dict(products=sub, start_cost=int(trace[0]),
                                     cost=int(cost), sweeps=(len(trace) - 1) // 4,
                                     trace=[int(x) for x in trace],
                                     plan_sha=plan_sha(plan.setup_m, plan.setup_r),
                                     final_sm=np.packbits(plan.setup_m, axis=1).tolist(),
                                     final_sr=np.packbits(plan.setup_r, axis=1).tolist(),
                                     wall_s=time.time() - t0)
    print("T520 sample", cost, (len(trace) - 1) // 4, time.time() - t0)
    with open(os.path.join(HERE, "big.json"), "w") as f:
        json.dump(out, f)


def gen_rng():
    data = {}
    triples = [(0, 0, 0), (0, 0, 1), (0, 5, 0), (7, 5, 0), (1, 3, 2), (9, 24, 1),
               (2**32 + 5, 1, 1), (2**64 - 1, 2**33, 1023), (123456789, 0, 511),
               (0, 1, 1023)]
    data["triples"] = np.array([[t[0] & (2**64 - 1), t[1], t[2]] for t in triples],
                               dtype=np.uint64)
    for i, (s, r, w) in enumerate(triples):
        rng = _worker_rng(s, r, w)
        data[f"t{i}_key"] = np.array(rng.bit_generator.state["state"]["key"], np.uint64)
        data[f"t{i}_raw"] = rng.bit_generator.random_raw(9)
        rng = _worker_rng(s, r, w)
        picks = []
        for n, k in ((2, 1), (4, 4), (104000, 5), (12, 3), (10000, 7), (5, 5),
                     (2**33, 3), (10001, 5), (20000, 401)):
            picks.append(rng.choice(n, size=k, replace=False))
        data[f"t{i}_choice"] = np.concatenate(picks).astype(np.int64)
        for n in (0, 1, 2, 7, 300):
            arr = np.arange(n, dtype=np.int64) * 3 + 1
            rng.shuffle(arr)
            data[f"t{i}_shuffle{n}"] = arr
        data[f"t{i}_tail"] = rng.bit_generator.random_raw(3)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **data)


def gen_gvns_small():
    data = {}
    shake_cases = []
    # (instance seed, K, T, demand_max, ratio, plan kind, k, (seed, round, w))
    for ci, (iseed, K, T, dmax, ratio) in enumerate(
            [(0, 5, 8, 9, 0.6), (1, 30, 20, 9, 0.6), (2, 6, 8, 9, 0.6),
             (3, 4, 8, 9, 0.6), (8, 3, 6, 9, 0.6), (11, 1, 2, 5, 0.0),
             (12, 1, 1, 5, 0.0), (13, 2, 3, 9, 1.0)]):
        inst = random_instance(iseed, products=K, periods=T, demand_max=dmax,
                               return_ratio=ratio)
        if ci == 5:   # make_instance([[2, 3]]) analogue: tight, forces fallbacks
            inst = Instance(1, 2, [[2, 3]], [[0, 0]], [1000], [400], [100], [100])
        for k, v in inst_arrays(inst).items():
            data[f"s{ci}_{k}"] = v
        inc = initial_solution(inst)
        vp, _ = vnd(inst, inc)
        for pk, plan in enumerate((inc, vp)):
            for strength in (1, 2, 3, 5, 9):
                for (s, r, w) in ((0, 0, 0), (4, 3, 1), (2**40, 7, 5)):
                    sp = shake(inst, plan, strength, _worker_rng(s, r, w))
                    key = f"s{ci}_p{pk}_k{strength}_{s}_{r}_{w}"
                    data[key + "_sm"] = sp.setup_m
                    data[key + "_sr"] = sp.setup_r
                    shake_cases.append(key)
        # worker_round and gvns with round caps
        for W in (1, 2, 3):
            cfg = SolverConfig(t_max=1e9, k_max=3, workers=W, seed=7, max_rounds=6)
            for pk, plan in enumerate((inc, vp)):
                for strength in (1, 3):
                    wp, wc = worker_round(inst, plan, strength, cfg, round_index=5)
                    key = f"s{ci}_wr_W{W}_p{pk}_k{strength}"
                    data[key + "_sm"] = wp.setup_m
                    data[key + "_sr"] = wp.setup_r
                    data[key + "_cost"] = np.int64(wc)
            res = gvns(inst, cfg)
            key = f"s{ci}_gvns_W{W}"
            data[key + "_sm"] = res.plan.setup_m
            data[key + "_sr"] = res.plan.setup_r
            data[key + "_cost"] = np.int64(res.cost)
            data[key + "_rounds"] = np.int64(res.rounds)
            data[key + "_shakes"] = np.int64(res.shake_calls)
    data["shake_keys"] = np.array(shake_cases)
    np.savez_compressed(os.path.join(HERE, "gvns_small.npz"), **data)


def gen_gvns_k1000():
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    out = {}
    for W, R in ((2, 20), (16, 4), (2, 150)):
        cfg = SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=W, seed=0,
                           max_rounds=R, vnd_mode="product-parallel", parallelism=8)
        t0 = time.time()
        res = gvns(inst, cfg)
        out[f"W{W}_R{R}"] = dict(cost=int(res.cost), rounds=res.rounds,
                                 shake_calls=res.shake_calls,
                                 plan_sha=plan_sha(res.plan.setup_m, res.plan.setup_r),
                                 wall_s=time.time() - t0)
        print("gvns K1000", W, R, res.cost, time.time() - t0)
    with open(os.path.join(HERE, "gvns_k1000.json"), "w") as f:
        json.dump(out, f, indent=1)


def gen_oracle_optimal():
    """enumerate_optimal (reference oracle.py:19-44) on small instances."""
    from remlot import enumerate_optimal
    out = []
    for seed, K, T, dmax in ((0, 3, 5, 9), (1, 2, 6, 9), (2, 4, 4, 5), (3, 1, 8, 9),
                             (4, 2, 10, 9), (5, 2, 1, 3), (6, 3, 3, 0)):
        inst = random_instance(seed, products=K, periods=T, demand_max=dmax,
                               setup_cost_range=(200, 8000), holding_cost_range=(100, 500))
        cost, plan = enumerate_optimal(inst)
        out.append(dict(seed=seed, products=K, periods=T, demand_max=dmax, cost=int(cost),
                        sm=plan.setup_m.astype(int).tolist(), sr=plan.setup_r.astype(int).tolist()))
    with open(os.path.join(HERE, "oracle_optimal.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    _kernels.warm_up()
    if "--oracle-only" in sys.argv:
        gen_oracle_optimal()
        sys.exit(0)
    if "--gvns-k1000-only" in sys.argv:
        gen_gvns_k1000()
        sys.exit(0)
    gen_instances()
    gen_rng()
    gen_small_cases()
    gen_c1()
    gen_k1000()
    gen_gvns_small()
    gen_gvns_k1000()
    gen_oracle_optimal()
    if "--big" in sys.argv:
        gen_big()

