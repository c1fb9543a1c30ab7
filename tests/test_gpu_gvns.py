"""Device shaking / worker rounds / GVNS vs the live reference's outputs
(tests/golden/gvns_small.npz, gvns_k1000.json) and the numpy RNG
restatement (oracle/numpy_rng.py, itself pinned to numpy)."""

import hashlib
import json
import os

import numpy as np
import pytest

import numpy_rng
from conftest import GOLDEN, GoldInstance, golden
from paper_1704_05132_b200 import (GeneratorConfig, Instance, SetupPlan, SolverConfig,
                                   generate_instance, gvns, initial_solution, shake, vnd,
                                   worker_round)
from paper_1704_05132_b200._native import rng_probe
from paper_1704_05132_b200.gvns import _worker_rng

pytestmark = pytest.mark.gpu


def _inst(data, prefix):
    g = GoldInstance(data, prefix)
    return Instance(g.products, g.periods, g.demand, g.returns, g.setup_cost_m,
                    g.setup_cost_r, g.holding_cost_m, g.holding_cost_r, g.unit_cost_m,
                    g.unit_cost_r)


def _plan_sha(plan):
    h = hashlib.sha256()
    h.update(np.packbits(plan.setup_m).tobytes())
    h.update(np.packbits(plan.setup_r).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("triple", [(0, 0, 0), (7, 5, 0), (2**32 + 5, 1, 1),
                                    (2**64 - 1, 2**33, 1023), (123456789, 0, 511)])
@pytest.mark.parametrize("pop,size,shuf", [(104000, 5, 0), (2, 1, 7), (12, 3, 300),
                                           (20000, 401, 2), (2**33, 3, 1), (10001, 5, 0)])
def test_device_philox_matches_numpy(triple, pop, size, shuf):
    raw, pick, sh, tail = rng_probe(*triple, pop, size, shuf)
    ref = numpy_rng.Philox.from_entropy(triple)
    assert raw.tolist() == [ref.next64() for _ in range(4)]
    assert pick.tolist() == ref.choice_noreplace(pop, size)
    arr = [3 * i + 1 for i in range(shuf)]
    ref.shuffle(arr)
    assert sh.tolist() == arr
    assert tail.tolist() == [ref.next64()]


def test_device_philox_matches_live_numpy_choice():
    for w in range(8):
        rng = _worker_rng(0, 3, w)
        rng.bit_generator.random_raw(4)   # the probe draws 4 raw words first
        want = rng.choice(104000, size=5, replace=False).tolist()
        assert rng_probe(0, 3, w, 104000, 5, 0)[1].tolist() == want


def _small_cases():
    data = golden("gvns_small.npz")
    cases = sorted({k.split("_")[0] for k in data.files if k.startswith("s")
                    and k.split("_")[0][1:].isdigit()})
    return data, cases


def test_public_shake_matches_reference():
    data, cases = _small_cases()
    n = 0
    for key in data["shake_keys"].tolist():
        ci, pk, kk, s, r, w = key.split("_")
        inst = _inst(data, ci + "_")
        inc = initial_solution(inst)
        plan = inc if pk == "p0" else vnd(inst, inc)[0]
        got = shake(inst, plan, int(kk[1:]), _worker_rng(int(s), int(r), int(w)))
        assert np.array_equal(got.setup_m, data[key + "_sm"]), key
        assert np.array_equal(got.setup_r, data[key + "_sr"]), key
        n += 1
    assert n > 100


def test_worker_round_matches_reference():
    data, cases = _small_cases()
    for ci in cases:
        inst = _inst(data, ci + "_")
        inc = initial_solution(inst)
        plans = (inc, vnd(inst, inc)[0])
        for W in (1, 2, 3):
            cfg = SolverConfig(t_max=1e9, k_max=3, workers=W, seed=7, max_rounds=6)
            for pk, plan in enumerate(plans):
                for k in (1, 3):
                    key = f"{ci}_wr_W{W}_p{pk}_k{k}"
                    got, cost = worker_round(inst, plan, k, cfg, round_index=5)
                    assert cost == int(data[key + "_cost"]), key
                    assert np.array_equal(got.setup_m, data[key + "_sm"]), key
                    assert np.array_equal(got.setup_r, data[key + "_sr"]), key


def test_gvns_round_capped_matches_reference():
    data, cases = _small_cases()
    for ci in cases:
        inst = _inst(data, ci + "_")
        for W in (1, 2, 3):
            cfg = SolverConfig(t_max=1e9, k_max=3, workers=W, seed=7, max_rounds=6)
            res = gvns(inst, cfg)
            key = f"{ci}_gvns_W{W}"
            assert res.cost == int(data[key + "_cost"]), key
            assert res.rounds == int(data[key + "_rounds"])
            assert res.shake_calls == int(data[key + "_shakes"])
            assert np.array_equal(res.plan.setup_m, data[key + "_sm"]), key
            assert np.array_equal(res.plan.setup_r, data[key + "_sr"]), key


@pytest.mark.parametrize("batch", ["1", "2", "5", "32"])
def test_gvns_speculative_batches_match_reference(batch, monkeypatch):
    """Speculative batches of rounds (rl_gvns_run) reproduce the sequential
    trajectory whatever the batch size: rounds accepted mid-batch discard the
    rest of the batch (round-capped goldens of the live reference)."""
    monkeypatch.setenv("RL_GVNS_BATCH", batch)
    data, cases = _small_cases()
    for ci in cases:
        inst = _inst(data, ci + "_")
        for W in (1, 3):
            cfg = SolverConfig(t_max=1e9, k_max=3, workers=W, seed=7, max_rounds=6)
            res = gvns(inst, cfg)
            key = f"{ci}_gvns_W{W}"
            assert res.cost == int(data[key + "_cost"]), key
            assert res.rounds == int(data[key + "_rounds"])
            assert np.array_equal(res.plan.setup_m, data[key + "_sm"]), key
            assert np.array_equal(res.plan.setup_r, data[key + "_sr"]), key
    with open(os.path.join(GOLDEN, "gvns_k1000.json")) as f:
        gold = json.load(f)
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    for name, R in (("W2_R20", 20), ("W2_R150", 150)):
        cfg = SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=2, seed=0, max_rounds=R)
        res = gvns(inst, cfg)
        g = gold[name]
        assert res.cost == g["cost"] and res.rounds == R, name
        assert res.shake_calls == g["shake_calls"]
        assert _plan_sha(res.plan) == g["plan_sha"], name


def test_gvns_k1000_matches_reference():
    """BASELINE config 2 (K=1000, T=52, full GVNS): round-capped runs of the
    live reference (W=2 x 20 rounds, W=16 x 4 rounds)."""
    with open(os.path.join(GOLDEN, "gvns_k1000.json")) as f:
        gold = json.load(f)
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    for name, (W, R) in (("W2_R20", (2, 20)), ("W16_R4", (16, 4))):
        cfg = SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=W, seed=0, max_rounds=R)
        res = gvns(inst, cfg)
        g = gold[name]
        assert res.cost == g["cost"], name
        assert res.rounds == g["rounds"] and res.shake_calls == g["shake_calls"]
        assert _plan_sha(res.plan) == g["plan_sha"], name


@pytest.mark.parametrize("batch", [None, 1, 3])
def test_sharded_replicas_device_backend_single_rank(batch):
    """The replica-sharded driver on the device backend (local speculative
    batches, candidate export, NCCL all-gather/broadcast, import) reproduces
    the reference's K=1000 W=16 GVNS and the W=128 x 4 replica golden with
    one rank, whatever the batch size; multi-rank splits are covered on
    gloo."""
    import socket

    import torch
    import torch.distributed as dist
    from paper_1704_05132_b200.sharded import sharded_gvns

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        with open(os.path.join(GOLDEN, "gvns_k1000.json")) as f:
            g = json.load(f)["W16_R4"]
        inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
        cfg = SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=16, seed=0, max_rounds=4)
        res = sharded_gvns(inst, cfg, batch=batch)
        assert res.cost == g["cost"] and res.rounds == 4 and res.shake_calls == 64
        assert _plan_sha(res.plan) == g["plan_sha"]
        with open(os.path.join(GOLDEN, "gvns_c5.json")) as f:
            g5 = json.load(f)["W128_R4"]
        cfg = SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=128, seed=0, max_rounds=4)
        res = sharded_gvns(inst, cfg, batch=batch)
        assert res.cost == g5["cost"] and res.rounds == 4
        assert _plan_sha(res.plan) == g5["plan_sha"]
    finally:
        dist.destroy_process_group()


def test_gvns_time_budget_follows_the_round_capped_trajectory():
    """A wall-clock-limited run (gvns.py:199-202: clock checked between
    rounds; here between in-flight speculative batches) stops near t_max and
    its result is the round-capped run with the same round count: the
    speculative batches never change the trajectory."""
    import time
    from paper_1704_05132_b200 import evaluate
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    t0 = time.monotonic()
    res = gvns(inst, SolverConfig(t_max=0.3, k_max=5, k_vnd_max=4, workers=2, seed=0))
    assert time.monotonic() - t0 < 5.0
    assert res.rounds > 0 and res.shake_calls == 2 * res.rounds
    assert evaluate(inst, res.plan) == res.cost
    capped = gvns(inst, SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=2, seed=0,
                                     max_rounds=res.rounds))
    assert capped.rounds == res.rounds and capped.cost == res.cost
    assert _plan_sha(capped.plan) == _plan_sha(res.plan)


def test_gvns_graph_replay_across_runs_on_one_handle():
    """rl_gvns_run's captured graph is rebuilt when the run's arguments
    change: runs with another seed, another round cap and the golden's again
    on the same cached device handle reproduce the golden."""
    with open(os.path.join(GOLDEN, "gvns_k1000.json")) as f:
        g = json.load(f)["W2_R20"]
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    base = dict(t_max=1e9, k_max=5, k_vnd_max=4, workers=2)
    other = gvns(inst, SolverConfig(seed=3, max_rounds=20, **base))
    assert other.rounds == 20
    gvns(inst, SolverConfig(seed=0, max_rounds=7, **base))
    res = gvns(inst, SolverConfig(seed=0, max_rounds=20, **base))
    assert res.cost == g["cost"] and _plan_sha(res.plan) == g["plan_sha"]


def test_gvns_zero_rounds_and_spent_budget_return_the_start():
    """gvns.py:200-206: the loop checks the budget and the round cap before
    the first round -- max_rounds=0 or a budget already spent gives the
    lot-for-lot start with 0 rounds (the device-resident loop is not
    entered)."""
    from paper_1704_05132_b200 import evaluate
    inst = generate_instance(GeneratorConfig(products=50, periods=52, seed=4))
    init = initial_solution(inst)
    for cfg in (SolverConfig(t_max=1e9, workers=2, seed=0, max_rounds=0),
                SolverConfig(t_max=1e-9, workers=2, seed=0)):
        res = gvns(inst, cfg)
        assert res.rounds == 0 and res.shake_calls == 0
        assert res.cost == evaluate(inst, init)
        assert np.array_equal(res.plan.setup_m, init.setup_m)
        assert np.array_equal(res.plan.setup_r, init.setup_r)


def test_gvns_device_loop_replays_with_new_caps():
    """The device loop's graph is built once per begin and replayed with the
    round cap read from device memory: consecutive capped runs on one
    Instance match the reference's round-capped goldens (gvns_k1000.json)."""
    with open(os.path.join(GOLDEN, "gvns_k1000.json")) as f:
        gold = json.load(f)
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    for name, R in (("W2_R150", 150), ("W2_R20", 20), ("W2_R150", 150)):
        res = gvns(inst, SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=2, seed=0,
                                      max_rounds=R))
        assert res.rounds == R and res.cost == gold[name]["cost"]
        assert _plan_sha(res.plan) == gold[name]["plan_sha"]
