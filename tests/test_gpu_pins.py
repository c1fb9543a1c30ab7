"""Round-2 parity pins at the BASELINE configs round 1 left unpinned
(fixtures: tests/golden/gen_pins_r02.py, from the live reference's generator
and gvns, and the C oracle pinned to the live reference):

* C4  K=10,000 T=520: the full descent -- cost, 1,605-entry trace, plan and
  per-product cost hashes, reference-equivalent evaluations, sweeps;
* C5  K=1,000 T=52 GVNS with W=128 x 4 and W=1,024 x 2 rounds (live
  reference gvns, gvns.py:184-221);
* the N=2 weak-scaling instance of bench.py (K=200,000 T=52): both ranks'
  shards descended on the device and merged like sharded.combine;
* the int64-cost and int64-value paths at K=10,000, and the forced-int64
  variant at C3 (K=100,000).
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1704_05132_b200 import (GeneratorConfig, SolverConfig, generate_instance, gvns,
                                   initial_solution)
from paper_1704_05132_b200._native import DeviceInstance
from paper_1704_05132_b200.sharded import merge_shards, shard_bounds

pytestmark = pytest.mark.gpu


def _load(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    with open(path) as f:
        return json.load(f)


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _plan_sha(sm, sr):
    return _sha(np.packbits(np.asarray(sm, bool)), np.packbits(np.asarray(sr, bool)))


def _cfg(g):
    return GeneratorConfig(products=g["products"], periods=g["periods"], seed=g["seed"],
                           demand_max=g["demand_max"],
                           setup_cost_range=tuple(g["setup_cost_range"]),
                           holding_cost_range=tuple(g["holding_cost_range"]),
                           unit_cost_range=tuple(g["unit_cost_range"]))


def _check_descent(g, variant=0, value_bytes=None, cost_bytes=None):
    inst = generate_instance(_cfg(g))
    assert _sha(inst.demand, inst.returns) == g["instance_sha"]
    start = initial_solution(inst)
    assert _plan_sha(start.setup_m, start.setup_r) == g["start_plan_sha"]
    dev = DeviceInstance(inst)
    if variant:
        dev.set_variant(variant)
    if value_bytes is not None:
        assert dev.info["value_bytes"] == value_bytes
    if cost_bytes is not None:
        assert dev.info["cost_bytes"] == cost_bytes
    sm, sr, trace, st = dev.vnd(start.setup_m, start.setup_r)
    assert st["start_cost"] == g["start_cost"]
    assert st["cost"] == g["cost"]
    assert trace.tolist() == g["trace"]
    assert st["sweeps"] == g["sweeps"]
    assert st["evals_reference"] == g["evals"]
    assert st["moves"] == g["moves"]
    assert _plan_sha(sm, sr) == g["plan_sha"]
    assert _sha(dev.product_costs(sm, sr)) == g["product_costs_sha"]
    return dev, st


@pytest.mark.parametrize("variant", [0, 2])
def test_c4_full_descent_matches_oracle(variant):
    """BASELINE config 4 in full: 463,359,284,884 after 401 sweeps."""
    g = _load("c4_full.json")
    assert g["cost"] == 463359284884 and len(g["trace"]) == 1605
    _check_descent(g, variant)


def test_int64_costs_path_k10000():
    """int32 values, costs beyond the int32 proof -> int64 cost arithmetic."""
    _check_descent(_load("int64_k10000.json")["v32_c64"], value_bytes=4, cost_bytes=8)


def test_int64_values_path_k10000():
    """sum D + sum R beyond 2^28 -> int64 values and costs."""
    _check_descent(_load("int64_k10000.json")["v64_c64"], value_bytes=8, cost_bytes=8)


def test_c3_forced_int64_variant_matches_golden():
    """Variant bit 4 runs C3 on the general int64 path: same result as the
    live reference (cost 449,100,704,810, trace and plan hash)."""
    with open(os.path.join(GOLDEN, "big.json")) as f:
        g = json.load(f)["k100000_t52"]
    inst = generate_instance(GeneratorConfig(products=100000, periods=52, seed=0))
    start = initial_solution(inst)
    dev = DeviceInstance(inst)
    dev.set_variant(16)
    assert dev.info["value_bytes"] == 8 and dev.info["cost_bytes"] == 8
    sm, sr, trace, st = dev.vnd(start.setup_m, start.setup_r)
    assert st["cost"] == g["cost"] == 449100704810
    assert trace.tolist() == g["trace"]
    assert _plan_sha(sm, sr) == g["plan_sha"]
    dev.set_variant(0)
    assert dev.info["value_bytes"] == 4 and dev.info["cost_bytes"] == 4


def test_n2_weak_scaling_instance_matches_oracle():
    """bench.py --gpus 2 (weak): rank r owns products [r*1e5, (r+1)*1e5) of
    the seed-0 K=200,000 instance, drawn on the device; the merged trace,
    cost and lockstep evaluation count equal the unsharded oracle descent."""
    g = _load("n2_weak.json")
    K, T = g["products"], g["periods"]
    cfg = GeneratorConfig(products=K, periods=T, seed=0)
    parts = []
    for r in range(2):
        lo, hi = shard_bounds(K, r, 2)
        dev = DeviceInstance.generate(cfg, lo, hi)
        sm, sr = dev.initial_solution()
        _, _, trace, st = dev.vnd(sm, sr)
        parts.append((trace.tolist(), dict(st, k_max=4)))
    g_trace, tot = merge_shards(parts, 4)
    assert tot["cost"] == g["cost"]
    assert g_trace == g["trace"]
    assert tot["evals_reference"] == g["evals"]
    assert tot["sweeps"] == g["sweeps"] and tot["moves"] == g["moves"]


@pytest.mark.parametrize("name,W,R", [("W128_R4", 128, 4), ("W1024_R2", 1024, 2)])
def test_c5_replicas_match_reference(name, W, R):
    """BASELINE config 5: 1,024 multi-start replicas (and 128, one GPU's
    share of 8) of K=1,000 T=52 -- round-capped live-reference gvns."""
    gold = _load("gvns_c5.json")
    if name not in gold:
        pytest.skip(f"{name} not generated")
    g = gold[name]
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    res = gvns(inst, SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=W, seed=0,
                                  max_rounds=R))
    assert res.cost == g["cost"] and res.rounds == R and res.shake_calls == g["shake_calls"]
    assert _plan_sha(res.plan.setup_m, res.plan.setup_r) == g["plan_sha"]


@pytest.mark.parametrize("name", ["K40_T100_W2_R30", "K16_T300_W3_R12", "K12_T520_W2_R8",
                                  "K20_T100_c64_W2_R10"])
def test_gvns_long_horizons_match_reference(name):
    """Round-capped live-reference gvns past the register rows (T = 100,
    300, 520: the device shake's multi-word rows and the shared-memory-row
    VND tasks) and with int64 costs (setup costs 5e7-2e8)."""
    g = _load("gvns_long.json")[name]
    inst = generate_instance(GeneratorConfig(products=g["products"], periods=g["periods"],
                                             seed=g["seed"],
                                             setup_cost_range=tuple(g["setup_cost_range"])))
    assert _sha(inst.demand, inst.returns) == g["instance_sha"]
    res = gvns(inst, SolverConfig(t_max=1e9, k_max=5, k_vnd_max=4, workers=g["workers"], seed=5,
                                  max_rounds=g["rounds"]))
    assert res.cost == g["cost"]
    assert res.rounds == g["rounds_done"] and res.shake_calls == g["shake_calls"]
    assert _plan_sha(res.plan.setup_m, res.plan.setup_r) == g["plan_sha"]
