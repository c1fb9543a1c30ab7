"""The reference package's own test expectations, run against this package.

Each test restates a behaviour the reference pins in pkg/tests (test_plan.py,
test_vnd.py, test_gvns.py) -- golden values, enumeration order, tie rules,
stale-move detection, mode independence, trace shape, shaking invariants --
and checks it on the CUDA path.  Independent costs come from the CPU oracle
(oracle/remlot_oracle.c, pinned to the live reference)."""

import numpy as np
import pytest

import oracle
from paper_1704_05132_b200 import (INFEASIBLE, MODE_PRODUCT_PARALLEL, MODE_SERIAL,
                                   SCHEME_HYBRID, SCHEME_PRODUCT_PARALLEL, SCHEME_SERIAL_VND,
                                   GeneratorConfig, Instance, SetupPlan, SolverConfig,
                                   apply_delta, best_neighbor, decode, enumerate_neighbors,
                                   evaluate, evaluate_product, generate_instance, gvns,
                                   initial_solution, next_strength, shake, solve_scheme, vnd,
                                   vnd_pass, worker_round)
from paper_1704_05132_b200.gvns import _worker_rng

pytestmark = pytest.mark.gpu


def make_instance(demand, returns=None, setup_m=1000, setup_r=400, holding_m=100,
                  holding_r=100, unit_m=0, unit_r=0):
    demand = np.asarray(demand, dtype=np.int64)
    K = demand.shape[0]
    if returns is None:
        returns = np.zeros_like(demand)
    rep = lambda x: np.full(K, x, dtype=np.int64)
    return Instance(K, demand.shape[1], demand, returns, rep(setup_m), rep(setup_r),
                    rep(holding_m), rep(holding_r), rep(unit_m), rep(unit_r))


def random_instance(seed, products=3, periods=6, demand_max=9, return_ratio=0.6):
    return generate_instance(GeneratorConfig(products=products, periods=periods,
                                             demand_max=demand_max, return_ratio=return_ratio,
                                             seed=seed))


def random_plan(inst, rng, density=0.4):
    K, T = inst.products, inst.periods
    return SetupPlan(rng.random((K, T)) < density, rng.random((K, T)) < density)


def feasible_plan(inst, rng):
    K, T = inst.products, inst.periods
    return SetupPlan(np.ones((K, T), dtype=bool), rng.random((K, T)) < 0.4)


def ref_cost(inst, plan):
    return oracle.evaluate(inst, plan.setup_m, plan.setup_r)


@pytest.fixture
def tiny():
    return make_instance([[2, 3]])


# ---- plan (reference test_plan.py) -------------------------------------

def test_golden_costs_and_decode(tiny):
    plan = SetupPlan([[True, False]], [[False, False]])
    assert evaluate(tiny, plan) == 1300
    d = decode(tiny, plan)
    assert d.total_cost == 1300
    assert d.qty_m.tolist() == [[5, 0]] and d.inv_m.tolist() == [[3, 0]]
    inst = make_instance([[2, 3]], returns=[[5, 0]])
    d = decode(inst, SetupPlan([[False, False]], [[True, False]]))
    assert d.total_cost == 700 and d.qty_r.tolist() == [[5, 0]]
    assert evaluate(make_instance([[0, 0, 0]]), SetupPlan.all_false(1, 3)) == 0
    assert evaluate(tiny, SetupPlan([[False, True]], [[False, False]])) == INFEASIBLE
    d = decode(make_instance([[0, 5]], returns=[[7, 0]]), SetupPlan.all_false(1, 2))
    assert d.total_cost == INFEASIBLE and not d.inv_r.any()
    assert d.to_csv().splitlines()[0] == "product,period,x_m,x_r,y_m,y_r"


def test_evaluate_matches_oracle_on_random_plans():
    rng = np.random.default_rng(0)
    for seed in range(30):
        inst = random_instance(seed)
        for density in (0.2, 0.5, 0.9):
            plan = random_plan(inst, rng, density)
            assert evaluate(inst, plan) == ref_cost(inst, plan)


def test_flow_balance_and_per_product():
    rng = np.random.default_rng(2)
    for seed in range(20):
        inst = random_instance(seed, products=4, periods=8)
        for plan in (initial_solution(inst),
                     SetupPlan(np.ones((4, 8), bool), rng.random((4, 8)) < 0.5)):
            d = decode(inst, plan)
            assert d.total_cost != INFEASIBLE
            pm = np.zeros(4, np.int64)
            pr = np.zeros(4, np.int64)
            for t in range(8):
                assert (d.inv_m[:, t] == pm + d.qty_m[:, t] + d.qty_r[:, t] - inst.demand[:, t]).all()
                assert (d.inv_r[:, t] == pr + inst.returns[:, t] - d.qty_r[:, t]).all()
                pm, pr = d.inv_m[:, t], d.inv_r[:, t]
            assert [evaluate_product(inst, plan, k) for k in range(4)] == d.cost_per_product.tolist()


def test_setup_charged_only_for_positive_quantity_and_errors(tiny):
    assert evaluate(tiny, SetupPlan([[True, False]], [[True, False]])) == 1300
    with pytest.raises(IndexError):
        evaluate_product(tiny, SetupPlan([[True, False]], [[False, False]]), 1)
    with pytest.raises(ValueError):
        evaluate(tiny, SetupPlan.all_false(2, 2))


def test_initial_solution_examples(tiny):
    p = initial_solution(tiny)
    assert p.setup_m.tolist() == [[True, True]] and p.setup_r.tolist() == [[False, False]]
    p = initial_solution(make_instance([[4, 4]], returns=[[3, 0]]))
    assert p.setup_r.tolist() == [[True, False]] and p.setup_m.tolist() == [[True, True]]
    for seed in range(25):
        inst = random_instance(seed, products=5, periods=9, return_ratio=1.0)
        assert evaluate(inst, initial_solution(inst)) != INFEASIBLE


# ---- vnd (reference test_vnd.py) ---------------------------------------

def test_enumeration_order_and_counts():
    plan = SetupPlan([[True, False, False]], [[False, False, False]])
    moves = enumerate_neighbors(plan, 1, 0)
    assert [m.periods for m in moves] == [(0,), (1,), (2,)]
    assert moves[0].new_m == (False,) and moves[1].new_m == (True,)
    plan = SetupPlan([[False, True, False]], [[True, True, False]])
    moves = enumerate_neighbors(plan, 3, 0)
    assert len(moves) == 3
    assert moves[0].periods == (1, 0) and moves[0].new_m == (False, True)
    assert moves[1].periods == (1, 2)
    assert moves[2].new_r == (False, True) and moves[2].periods == (1, 2)
    assert enumerate_neighbors(SetupPlan.all_false(1, 4), 3, 0) == []
    one = enumerate_neighbors(SetupPlan([[True, False]], [[False, False]]), 4, 0)
    assert len(one) == 1 and one[0].new_m == (False,) and one[0].new_r == (True,)
    with pytest.raises(ValueError):
        enumerate_neighbors(plan, 5, 0)
    with pytest.raises(IndexError):
        enumerate_neighbors(plan, 1, 3)


def test_move_apply_invert_and_stale():
    rng = np.random.default_rng(3)
    for seed in range(6):
        inst = random_instance(seed, products=3, periods=6)
        plan = random_plan(inst, rng, 0.5)
        for nbh in (1, 2, 3, 4):
            for k in range(3):
                for move in enumerate_neighbors(plan, nbh, k):
                    changed = move.apply(plan)
                    assert changed != plan and move.inverted().apply(changed) == plan
    plan = SetupPlan([[True, False]], [[False, False]])
    move = enumerate_neighbors(plan, 1, 0)[0]
    with pytest.raises(ValueError, match="stale"):
        move.apply(SetupPlan([[False, False]], [[False, False]]))


def test_best_neighbor_golden_and_bruteforce(tiny):
    found = best_neighbor(tiny, SetupPlan([[True, True]], [[False, False]]), 1, 0)
    assert found is not None and found[1] == 700
    assert found[0].periods == (1,) and found[0].new_m == (False,)
    assert best_neighbor(tiny, SetupPlan([[True, False]], [[False, False]]), 1, 0) is None
    assert best_neighbor(make_instance([[5]]), SetupPlan([[True]], [[False]]), 1, 0) is None
    rng = np.random.default_rng(4)
    for seed in range(8):
        inst = random_instance(seed, products=2, periods=6)
        plan = feasible_plan(inst, rng)
        for nbh in (1, 2, 3, 4):
            for k in range(2):
                base = ref_cost(inst, plan)
                moves = enumerate_neighbors(plan, nbh, k)
                best_cost, best_idx = base, None
                for i, m in enumerate(moves):
                    c = ref_cost(inst, m.apply(plan))
                    if c < best_cost:
                        best_cost, best_idx = c, i
                found = best_neighbor(inst, plan, nbh, k)
                if best_idx is None:
                    assert found is None
                else:
                    assert found[0] == moves[best_idx] and found[1] == base - best_cost


def test_vnd_pass_and_apply_delta():
    inst = make_instance([[2, 3], [2, 3]])
    plan = SetupPlan([[True, True], [True, True]], np.zeros((2, 2), dtype=bool))
    delta = vnd_pass(inst, plan, 1)
    assert delta.diff == 1400 and delta.decreases == (700, 700)
    with pytest.raises(ValueError, match="stale"):
        apply_delta(SetupPlan(~plan.setup_m, plan.setup_r), delta)
    rng = np.random.default_rng(6)
    for seed in range(15):
        inst = random_instance(seed, products=5, periods=7)
        plan = feasible_plan(inst, rng)
        for nbh in (1, 2, 3, 4):
            d = vnd_pass(inst, plan, nbh)
            assert evaluate(inst, apply_delta(plan, d)) == evaluate(inst, plan) - d.diff
            assert vnd_pass(inst, plan, nbh, mode=MODE_PRODUCT_PARALLEL, parallelism=8) == d
    with pytest.raises(ValueError):
        vnd_pass(inst, plan, 1, mode="gpu")


def test_vnd_examples_trace_and_composition(tiny):
    plan, cost = vnd(tiny, SetupPlan([[True, True]], [[False, False]]))
    assert cost == 1300 and plan.setup_m.tolist() == [[True, False]]
    start = SetupPlan([[True, False]], [[False, False]])
    assert vnd(tiny, start) == (start, 1300)
    for bad in (0, 5):
        with pytest.raises(ValueError):
            vnd(tiny, start, k_max=bad)
    rng = np.random.default_rng(10)
    for seed in range(6):
        inst = random_instance(seed, products=4, periods=8)
        start = feasible_plan(inst, rng)
        exp_plan, exp_cost = start, evaluate(inst, start)
        sweeps = 0
        while True:
            sweeps += 1
            improvement = False
            for nbh in (1, 2, 3, 4):
                d = vnd_pass(inst, exp_plan, nbh)
                if d.diff > 0:
                    exp_plan = apply_delta(exp_plan, d)
                    exp_cost -= d.diff
                    improvement = True
            if not improvement:
                break
        trace = []
        plan, cost = vnd(inst, start, trace=trace)
        assert (plan, cost) == (exp_plan, exp_cost)
        assert len(trace) == 1 + 4 * sweeps and trace[0] == evaluate(inst, start)
        assert all(a >= b for a, b in zip(trace, trace[1:])) and trace[-1] == cost
        for nbh in (1, 2, 3, 4):
            for k in range(4):
                assert best_neighbor(inst, plan, nbh, k) is None


# ---- gvns (reference test_gvns.py) -------------------------------------

def _hamming(a, b):
    return int((a.setup_m != b.setup_m).sum() + (a.setup_r != b.setup_r).sum())


def test_shake_invariants():
    inst = random_instance(0, products=5, periods=8)
    plan = initial_solution(inst)
    rng = np.random.default_rng(0)
    for _ in range(20):
        s = shake(inst, plan, 1, rng)
        assert _hamming(plan, s) == 1 and evaluate(inst, s) != INFEASIBLE
    tight = make_instance([[2, 3]])
    rng = np.random.default_rng(11)
    for strength in (1, 2, 3, 4, 100):
        for _ in range(10):
            assert evaluate(tight, shake(tight, initial_solution(tight), strength, rng)) != INFEASIBLE
    with pytest.raises(ValueError):
        shake(tight, initial_solution(tight), 0, np.random.default_rng(0))


def test_worker_round_semantics():
    inst = random_instance(4, products=4, periods=8)
    inc = initial_solution(inst)
    cfg = SolverConfig(t_max=10.0, k_max=3, workers=3, seed=2)
    plan, cost = worker_round(inst, inc, 2, cfg, round_index=1)
    cands = [vnd(inst, shake(inst, inc, 2, _worker_rng(2, 1, w))) for w in range(3)]
    assert cost == min(c for _, c in cands)
    assert plan == next(p for p, c in cands if c == cost)
    zero = make_instance([[0, 0, 0]])
    cfg = SolverConfig(t_max=10.0, k_max=3, workers=2, seed=3)
    plan, cost = worker_round(zero, initial_solution(zero), 2, cfg, round_index=0)
    assert cost == 0
    assert plan == vnd(zero, shake(zero, initial_solution(zero), 2, _worker_rng(3, 0, 0)))[0]


def test_gvns_determinism_and_counts():
    assert next_strength(2, True, 5) == 1 and next_strength(5, False, 5) == 1
    assert next_strength(2, False, 5) == 3
    inst = random_instance(6, products=4, periods=7)
    cfg = SolverConfig(t_max=1e9, max_rounds=25, workers=2, seed=9, k_max=3)
    a, b = gvns(inst, cfg), gvns(inst, cfg)
    assert (a.cost, a.plan, a.rounds) == (b.cost, b.plan, 25)
    assert a.shake_calls == 50
    assert a.cost <= evaluate(inst, initial_solution(inst))
    assert evaluate(inst, a.plan) == a.cost
    r = gvns(random_instance(5, products=3, periods=6), SolverConfig(t_max=1e-9, seed=1))
    assert r.rounds <= 1


def test_gvns_reaches_oracle_optimum():
    from paper_1704_05132_b200 import enumerate_optimal
    inst = random_instance(7, products=2, periods=5, demand_max=9)
    res = gvns(inst, SolverConfig(t_max=1e9, max_rounds=300, workers=2, seed=4, k_max=3))
    assert res.cost == enumerate_optimal(inst)[0]


def test_solve_scheme_dispatch():
    inst = random_instance(9, products=4, periods=8)
    r = solve_scheme(inst, SolverConfig(t_max=10.0, scheme=SCHEME_SERIAL_VND, seed=1))
    assert r.shake_calls == 0 and r.rounds == 0
    assert (r.plan, r.cost) == vnd(inst, initial_solution(inst))
    base = dict(t_max=1e9, max_rounds=4, workers=2, seed=5, k_max=3)
    h = solve_scheme(inst, SolverConfig(scheme=SCHEME_HYBRID, **base))
    assert h.shake_calls == 8
    p = solve_scheme(inst, SolverConfig(scheme=SCHEME_PRODUCT_PARALLEL, **base))
    assert p.shake_calls == p.rounds == 4
    m = solve_scheme(inst, SolverConfig(scheme="multiworker", vnd_mode=MODE_SERIAL, **base))
    assert (m.cost, m.plan) == (h.cost, h.plan)
    for bad in (dict(t_max=0), dict(t_max=1, k_max=0), dict(t_max=1, workers=0),
                dict(t_max=1, scheme="bogus"), dict(t_max=1, vnd_mode="gpu")):
        with pytest.raises(ValueError):
            SolverConfig(**bad)


# ---- oracle (reference oracle.py / test_oracle.py) ------------------------

def test_enumerate_optimal_matches_reference_goldens():
    import json
    import os
    from conftest import GOLDEN
    from paper_1704_05132_b200 import enumerate_optimal
    with open(os.path.join(GOLDEN, "oracle_optimal.json")) as f:
        gold = json.load(f)
    for g in gold:
        inst = generate_instance(GeneratorConfig(
            products=g["products"], periods=g["periods"], demand_max=g["demand_max"],
            return_ratio=0.6, setup_cost_range=(200, 8000), holding_cost_range=(100, 500),
            seed=g["seed"]))
        cost, plan = enumerate_optimal(inst)
        assert cost == g["cost"]
        assert plan.setup_m.astype(int).tolist() == g["sm"]
        assert plan.setup_r.astype(int).tolist() == g["sr"]
        assert evaluate(inst, plan) == cost


def test_enumerate_optimal_bounds_heuristics_and_refuses_long_horizons():
    from paper_1704_05132_b200 import enumerate_optimal
    for seed in range(5):
        inst = random_instance(100 + seed, products=3, periods=6)
        opt, plan = enumerate_optimal(inst)
        assert vnd(inst, initial_solution(inst))[1] >= opt
        assert evaluate(inst, plan) == opt
    with pytest.raises(ValueError):
        enumerate_optimal(random_instance(1, products=1, periods=11))
