"""Reentrancy of the drop-in boundary and device-state invalidation.

The reference's kernels are nogil and reentrant (reference _kernels.py:3-4):
its ``run_bench(parallel_cells=True)`` runs ``solve_scheme`` from 4 threads
on one Instance (bench.py:196-198) and SPEC.md:351 lets W worker threads nest
VND calls.  Here the C ABI serialises calls per handle and GVNS sessions get
their own handles (``_native.session``); results must equal the serial
goldens of the live reference.
"""

import hashlib
import json
import os
import threading

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, golden
from paper_1704_05132_b200 import (GeneratorConfig, Instance, SolverConfig, evaluate,
                                   generate_instance, gvns, initial_solution, vnd)
from paper_1704_05132_b200 import _native

pytestmark = pytest.mark.gpu


def _plan_sha(plan):
    h = hashlib.sha256()
    h.update(np.packbits(plan.setup_m).tobytes())
    h.update(np.packbits(plan.setup_r).tobytes())
    return h.hexdigest()


def _run_threads(fns):
    out = [None] * len(fns)
    errs = []

    def run(i, f):
        try:
            out[i] = f()
        except BaseException as e:   # noqa: BLE001 -- re-raised below
            errs.append(e)

    th = [threading.Thread(target=run, args=(i, f)) for i, f in enumerate(fns)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


def test_threads_share_one_instance_vnd_and_gvns():
    """4 threads x (vnd + gvns) on one Instance == the serial goldens
    (K=1000 T=52: vnd cost/plan of the live reference, gvns W=2 x 20)."""
    with open(os.path.join(GOLDEN, "gvns_k1000.json")) as f:
        g = json.load(f)["W2_R20"]
    k1000 = golden("k1000.npz")
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    start = initial_solution(inst)
    cfg = SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=2, seed=0, max_rounds=20)

    def work():
        res = []
        for _ in range(2):
            trace = []
            plan, cost = vnd(inst, start, trace=trace)
            res.append(("vnd", cost, plan.setup_m.copy(), plan.setup_r.copy(), trace))
            r = gvns(inst, cfg)
            res.append(("gvns", r.cost, r.rounds, _plan_sha(r.plan)))
        return res

    for res in _run_threads([work] * 4):
        for item in res:
            if item[0] == "vnd":
                _, cost, sm, sr, trace = item
                assert cost == int(k1000["cost"])
                assert np.array_equal(np.packbits(sm, axis=1), k1000["final_sm"])
                assert np.array_equal(np.packbits(sr, axis=1), k1000["final_sr"])
                assert trace == k1000["trace"].tolist()
            else:
                _, cost, rounds, sha = item
                assert (cost, rounds, sha) == (g["cost"], 20, g["plan_sha"])


def test_threads_on_separate_instances_overlap():
    """Threads on different instances (different handles) give each
    instance's own serial result."""
    insts = [generate_instance(GeneratorConfig(products=300, periods=52, seed=s))
             for s in range(4)]
    want = []
    for inst in insts:
        plan, cost = vnd(inst, initial_solution(inst))
        want.append((cost, _plan_sha(plan)))

    def job(inst):
        return lambda: [(lambda p: (p[1], _plan_sha(p[0])))(vnd(inst, initial_solution(inst)))
                        for _ in range(3)]

    for w, got in zip(want, _run_threads([job(i) for i in insts])):
        assert all(x == w for x in got)


def test_in_place_edit_invalidates_device_copy():
    """The reference re-reads the arrays on every call (its own
    test_model.py:173 edits a fresh instance in place): after an upload the
    arrays are read-only, and an edit made after re-enabling writes, or a
    reassigned field, is seen by the next call -- never a stale copy."""
    from paper_1704_05132_b200 import SetupPlan
    inst = generate_instance(GeneratorConfig(products=50, periods=52, seed=1))
    sm = np.zeros((50, 52), bool)
    sm[:, 0] = True   # everything produced in period 0: every demand is held
    plan = SetupPlan(sm, np.zeros((50, 52), bool))
    before = evaluate(inst, plan)
    with pytest.raises(ValueError):   # the uploaded arrays are read-only
        inst.demand[0, -1] += 7
    inst.demand.setflags(write=True)  # an explicit opt-in re-uploads
    inst.demand[0, -1] += 7
    got = evaluate(inst, plan)
    assert got == oracle.evaluate(inst, plan.setup_m, plan.setup_r)
    assert got - before == 7 * 51 * int(inst.holding_cost_m[0])
    inst.holding_cost_m = inst.holding_cost_m + 1   # reassignment
    assert evaluate(inst, plan) == oracle.evaluate(inst, plan.setup_m, plan.setup_r)


def test_update_to_wider_values_drops_gvns_state():
    """ADVICE r1 (gvns_impl.cuh:741): after rl_instance_update switches the
    value width, the handle's GVNS state (scratch sized for the old width,
    captured graph over freed rows) must be gone: rl_gvns_run without a new
    begin fails cleanly, and a fresh begin gives the oracle's VND image."""
    inst = generate_instance(GeneratorConfig(products=40, periods=52, seed=2))
    dev = _native.DeviceInstance(inst)
    assert dev.info["value_bytes"] == 4
    sm, sr = dev.initial_solution()
    dev.gvns_begin(2, 5, 4, 0, sm, sr, batch=2)
    dev.gvns_run(4)
    dev.gvns_run(8)   # captured graph
    big = Instance(inst.products, inst.periods, inst.demand * 10_000_000,
                   inst.returns * 10_000_000, inst.setup_cost_m, inst.setup_cost_r,
                   inst.holding_cost_m, inst.holding_cost_r)
    dev.update(big)
    assert dev.info["value_bytes"] == 8
    with pytest.raises(ValueError):
        dev.gvns_run(12)
    sm, sr = dev.initial_solution()
    cost = dev.gvns_begin(2, 5, 4, 0, sm, sr, batch=2)
    assert cost == oracle.evaluate(big, sm, sr)
    rounds = 0
    for _ in range(100):   # one speculative batch per call
        dev.gvns_run(12)
        rounds = dev.gvns_state(0, want_plan=False)[2]["rounds"]
        if rounds == 12:
            break
    assert rounds == 12


def test_fallback_slot_overflow_truncates_batch(monkeypatch):
    """ADVICE r1 (gvns_impl.cuh:764): speculative rounds share the fallback
    slots.  On K=1, T=1, D=5, R=0 every strength-2 shake falls back
    (gvns.py:124-137: both bits flipped is infeasible, the incumbent equals
    the lot-for-lot start).  With one round's worth of slots and batches of
    4 rounds the slots overflow; the batch is truncated and re-run instead
    of failing, and the trajectory is the sequential one (no round improves:
    the lot-for-lot plan, cost k_M)."""
    monkeypatch.setenv("RL_GVNS_FB_SLOTS", "3")
    monkeypatch.setenv("RL_GVNS_BATCH", "4")
    inst = Instance(1, 1, [[5]], [[0]], [1000], [400], [100], [100])
    res = gvns(inst, SolverConfig(t_max=1e9, k_max=2, k_vnd_max=4, workers=3, seed=0,
                                  max_rounds=10))
    assert res.rounds == 10 and res.shake_calls == 30
    assert res.cost == 1000
    assert res.plan.setup_m.tolist() == [[True]] and res.plan.setup_r.tolist() == [[False]]
