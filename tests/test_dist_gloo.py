"""Multi-rank host logic on CPU (gloo, world_size 2): product sharding and
the totals/trace combine of paper_1704_05132_b200.sharded, with the CPU
oracle as each rank's local descent, must equal one unsharded reference
descent bit for bit (trace, cost, plan, lockstep evaluation count)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import ROOT
from paper_1704_05132_b200.model import GeneratorConfig, generate_instance
from paper_1704_05132_b200.plan import SetupPlan
from paper_1704_05132_b200.sharded import shard_bounds, sharded_vnd


def _oracle_local_vnd(shard, sm, sr, k_max):
    m, r, cost, trace, st = oracle.vnd(shard, sm, sr, k_max)
    feas = oracle.product_costs(shard, m, r) != oracle.INFEASIBLE
    ntot = 0
    for k in np.flatnonzero(feas):
        for nbh in range(1, k_max + 1):
            ntot += len(oracle.list_moves(nbh, m[k], r[k])[0])
    return m, r, trace.tolist(), dict(evals=st["evals"], moves=st["moves"],
                                      evals_reference=st["evals"], ntot_sum=ntot)


def _worker(rank, world, port, cases, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        for K, T, seed, plan_kind in cases:
            inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=seed,
                                                     demand_max=30 if T < 20 else 100))
            if plan_kind == "init":
                sm, sr = oracle.initial_solution(inst)
            else:
                rng = np.random.default_rng(seed)
                sm, sr = rng.random((K, T)) < 0.5, rng.random((K, T)) < 0.5
            plan, cost, trace, tot = sharded_vnd(inst, SetupPlan(sm, sr), 4,
                                                 local_vnd=_oracle_local_vnd)
            res.append((cost, trace, tot["evals_reference"], tot["moves"], tot["sweeps"],
                        np.packbits(plan.setup_m).tobytes(), np.packbits(plan.setup_r).tobytes()))
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [(7, 9, 1, "init"), (13, 52, 0, "init"), (5, 6, 3, "random"), (1, 8, 4, "init")]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_vnd_equals_unsharded_reference(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, (K, T, seed, kind) in enumerate(CASES):
        inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=seed,
                                                 demand_max=30 if T < 20 else 100))
        if kind == "init":
            sm, sr = oracle.initial_solution(inst)
        else:
            rng = np.random.default_rng(seed)
            sm, sr = rng.random((K, T)) < 0.5, rng.random((K, T)) < 0.5
        m, r, cost, trace, st = oracle.vnd(inst, sm, sr)
        for rank in range(world):
            gcost, gtrace, gref, gmoves, gsweeps, pm, pr = got[rank][i]
            assert gcost == cost
            assert gtrace == trace.tolist()
            assert gref == st["evals"]
            assert gmoves == st["moves"] and gsweeps == st["sweeps"]
            assert pm == np.packbits(m).tobytes() and pr == np.packbits(r).tobytes()


def test_shard_bounds_cover_products_in_order():
    for K in (1, 5, 100000):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(K, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == K
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def _gvns_worker(rank, world, port, out_q, batch=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from gvns_oracle import OracleRounds
        from paper_1704_05132_b200.gvns import SolverConfig
        from paper_1704_05132_b200.model import Instance
        from paper_1704_05132_b200.sharded import sharded_gvns
        from conftest import GoldInstance, golden
        data = golden("gvns_small.npz")
        res = []
        for ci in ("s0", "s3", "s5", "s7"):
            g = GoldInstance(data, ci + "_")
            inst = Instance(g.products, g.periods, g.demand, g.returns, g.setup_cost_m,
                            g.setup_cost_r, g.holding_cost_m, g.holding_cost_r,
                            g.unit_cost_m, g.unit_cost_r)
            cfg = SolverConfig(t_max=1e9, k_max=3, workers=3, seed=7, max_rounds=6)
            r = sharded_gvns(inst, cfg, backend=OracleRounds(inst), batch=batch)
            res.append((ci, r.cost, r.rounds, r.shake_calls, r.plan.setup_m.tobytes(),
                        r.plan.setup_r.tobytes()))
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,batch", [(2, None), (3, None), (2, 1), (3, 5)])
def test_sharded_replicas_equal_reference_gvns(world, batch):
    """Workers split over ranks (BASELINE config 5 shape), speculative
    batches of rounds with one collective per batch: the cross-rank best-of
    join reproduces the reference gvns() (W=3, 6 rounds) exactly, whatever
    the batch size."""
    from conftest import golden
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gvns_worker, args=(r, world, port, q, batch))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    data = golden("gvns_small.npz")
    for rank in range(world):
        for ci, cost, rounds, shakes, pm, pr in got[rank]:
            key = f"{ci}_gvns_W3"
            assert cost == int(data[key + "_cost"]), key
            assert rounds == 6 and shakes == 18
            assert pm == data[key + "_sm"].tobytes() and pr == data[key + "_sr"].tobytes(), key


@pytest.mark.parametrize("world", [2, 3, 8])
def test_merge_shards_equals_unsharded_reference(world):
    """sharded.merge_shards (the combine of all shards in one process, used
    to pin multi-rank results on one device) == one unsharded descent."""
    from paper_1704_05132_b200.sharded import merge_shards
    for K, T, seed, kind in CASES:
        inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=seed,
                                                 demand_max=30 if T < 20 else 100))
        if kind == "init":
            sm, sr = oracle.initial_solution(inst)
        else:
            rng = np.random.default_rng(seed)
            sm, sr = rng.random((K, T)) < 0.5, rng.random((K, T)) < 0.5
        parts = []
        for r in range(world):
            lo, hi = shard_bounds(K, r, world)
            if hi > lo:
                _, _, trace, st = _oracle_local_vnd(inst.slice(lo, hi), sm[lo:hi], sr[lo:hi], 4)
                parts.append((trace, st))
        g_trace, tot = merge_shards(parts, 4)
        m, r_, cost, trace, st = oracle.vnd(inst, sm, sr)
        assert g_trace == trace.tolist() and tot["cost"] == cost
        assert tot["evals_reference"] == st["evals"] and tot["sweeps"] == st["sweeps"]
        assert tot["moves"] == st["moves"]


def _gvns_long_worker(rank, world, port, names, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import json
        from gvns_oracle import OracleRounds
        from conftest import GOLDEN
        from paper_1704_05132_b200.gvns import SolverConfig
        from paper_1704_05132_b200.sharded import sharded_gvns
        with open(os.path.join(GOLDEN, "gvns_long.json")) as f:
            gold = json.load(f)
        res = []
        for name in names:
            g = gold[name]
            inst = generate_instance(GeneratorConfig(
                products=g["products"], periods=g["periods"], seed=g["seed"],
                setup_cost_range=tuple(g["setup_cost_range"])))
            cfg = SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=g["workers"], seed=5,
                               max_rounds=g["rounds"])
            r = sharded_gvns(inst, cfg, backend=OracleRounds(inst))
            res.append((name, r.cost, r.rounds, r.shake_calls))
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_oracle_gvns_long_horizons_match_reference():
    """The CPU restatement of the shake / worker rounds (oracle/gvns_oracle.py)
    reproduces the live reference's round-capped gvns past the register rows
    (T = 100, with int32 and int64 costs; tests/golden/gvns_long.json), the
    workers split over 2 gloo ranks."""
    import json
    from conftest import GOLDEN
    names = ["K40_T100_W2_R30", "K20_T100_c64_W2_R10"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gvns_long_worker, args=(r, 2, port, names, q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    with open(os.path.join(GOLDEN, "gvns_long.json")) as f:
        gold = json.load(f)
    for rank in range(2):
        for name, cost, rounds, shakes in got[rank]:
            g = gold[name]
            assert cost == g["cost"], name
            assert rounds == g["rounds_done"] and shakes == g["shake_calls"], name
