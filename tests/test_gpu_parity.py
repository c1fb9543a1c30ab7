"""CUDA path vs the reference: golden fixtures made by the live reference
(tests/golden/) and the CPU oracle (oracle/), bit-exact integer equality.

Every call goes through the C ABI (libremlot_b200.so via ctypes)."""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, GoldInstance, golden
from paper_1704_05132_b200 import (GeneratorConfig, Instance, generate_instance,
                                   initial_solution)
from paper_1704_05132_b200._native import DeviceInstance, list_moves

pytestmark = pytest.mark.gpu
NAMES = ("dec", "p0", "m0", "r0", "p1", "m1", "r1")


def _inst(g):
    return Instance(g.products, g.periods, g.demand, g.returns, g.setup_cost_m,
                    g.setup_cost_r, g.holding_cost_m, g.holding_cost_r, g.unit_cost_m,
                    g.unit_cost_r)


def _plan_sha(sm, sr):
    h = hashlib.sha256()
    h.update(np.packbits(np.asarray(sm, bool)).tobytes())
    h.update(np.packbits(np.asarray(sr, bool)).tobytes())
    return h.hexdigest()


def _cases(small_cases):
    for idx, K, T in small_cases["cases"]:
        inst = _inst(GoldInstance(small_cases, f"c{idx}_"))
        dev = DeviceInstance(inst)
        for pi in range(int(small_cases["n_plans"])):
            yield inst, dev, f"c{idx}_{pi}_"


def test_product_costs_golden(small_cases):
    for inst, dev, p in _cases(small_cases):
        got = dev.product_costs(small_cases[p + "sm"], small_cases[p + "sr"])
        np.testing.assert_array_equal(got, small_cases[p + "cost"], err_msg=p)


def test_list_moves_golden(small_cases):
    for inst, dev, p in _cases(small_cases):
        sm, sr = small_cases[p + "sm"], small_cases[p + "sr"]
        for nbh in (1, 2, 3, 4):
            ns = small_cases[p + f"lm{nbh}_n"]
            for k in range(min(inst.products, 3)):
                got = list_moves(nbh, sm[k], sr[k])
                n = int(ns[k])
                assert len(got[0]) == n
                for name, g in zip(("mp0", "mm0", "mr0", "mp1", "mm1", "mr1"), got):
                    np.testing.assert_array_equal(g, small_cases[p + f"lm{nbh}_{name}"][k, :n])


def test_scan_products_golden(small_cases):
    for inst, dev, p in _cases(small_cases):
        for nbh in (1, 2, 3, 4):
            out, ev = dev.scan_products(small_cases[p + "sm"], small_cases[p + "sr"], nbh)
            dec = out[0]
            for name, g in zip(NAMES, out):
                g = np.array(g)
                if name in ("m0", "r0"):
                    g &= dec > 0
                if name in ("m1", "r1"):
                    g &= (dec > 0) & (out[4] >= 0)
                np.testing.assert_array_equal(g, small_cases[p + f"scan{nbh}_{name}"],
                                              err_msg=f"{p} nbh={nbh} {name}")
            _, oev = oracle.scan_products(inst, small_cases[p + "sm"], small_cases[p + "sr"], nbh)
            assert ev == oev


@pytest.mark.parametrize("variant", [8, 4, 64])
def test_vnd_golden(small_cases, variant):
    for inst, dev, p in _cases(small_cases):
        dev.set_variant(variant)
        for k_max in (1, 4):
            sm, sr, trace, st = dev.vnd(small_cases[p + "sm"], small_cases[p + "sr"], k_max)
            assert st["cost"] == int(small_cases[p + f"vnd{k_max}_cost"]), p
            np.testing.assert_array_equal(trace, small_cases[p + f"vnd{k_max}_trace"], err_msg=p)
            np.testing.assert_array_equal(sm, small_cases[p + f"vnd{k_max}_sm"], err_msg=p)
            np.testing.assert_array_equal(sr, small_cases[p + f"vnd{k_max}_sr"], err_msg=p)
            _, _, _, _, ost = oracle.vnd(inst, small_cases[p + "sm"], small_cases[p + "sr"], k_max)
            assert st["evals_reference"] == ost["evals"], p
            assert st["moves"] == ost["moves"] and st["sweeps"] == ost["sweeps"], p


def test_initial_solution_golden(small_cases):
    for inst, dev, p in _cases(small_cases):
        if p.endswith("_0_"):
            sm, sr = dev.initial_solution()
            np.testing.assert_array_equal(sm, small_cases[p + "sm"])
            np.testing.assert_array_equal(sr, small_cases[p + "sr"])


def test_decode_matches_oracle(small_cases):
    for inst, dev, p in _cases(small_cases):
        got = dev.decode(small_cases[p + "sm"], small_cases[p + "sr"])
        want = oracle.decode(inst, small_cases[p + "sm"], small_cases[p + "sr"])
        for g, w in zip(got, want):
            np.testing.assert_array_equal(g, w, err_msg=p)


def test_c1_every_lockstep_pass():
    """BASELINE config 1 (K=10, T=52, seed 0): all 180 passes of the
    reference trajectory, then the fused VND: cost 44,066,661."""
    g = golden("c1_trajectory.npz")
    inst = generate_instance(GeneratorConfig(products=10, periods=52, seed=0))
    dev = DeviceInstance(inst)
    sm, sr = g["start_sm"].copy(), g["start_sr"].copy()
    for i in range(g["pass_dec"].shape[0]):
        out, _ = dev.scan_products(sm, sr, i % 4 + 1)
        dec = out[0]
        for name, got in zip(NAMES, out):
            got = np.array(got)
            if name in ("m0", "r0"):
                got &= dec > 0
            if name in ("m1", "r1"):
                got &= (dec > 0) & (out[4] >= 0)
            np.testing.assert_array_equal(got, g["pass_" + name][i], err_msg=f"pass {i} {name}")
        sm, sr = sm.copy(), sr.copy()
        dev.apply_scan(out, sm, sr)
    np.testing.assert_array_equal(sm, g["final_sm"])
    fm, fr, trace, st = dev.vnd(g["start_sm"], g["start_sr"])
    assert st["cost"] == int(g["cost"]) == 44066661
    np.testing.assert_array_equal(trace, g["trace"])
    np.testing.assert_array_equal(fm, g["final_sm"])
    np.testing.assert_array_equal(fr, g["final_sr"])
    assert st["evals_reference"] == int(g["evals"]) == 70890
    assert st["moves"] == int(g["moves"]) == 738
    assert st["sweeps"] == int(g["sweeps"]) == 45


@pytest.mark.parametrize("variant", [8, 4, 64])
def test_k1000_vnd_golden(variant):
    g = golden("k1000.npz")
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    start = initial_solution(inst)
    np.testing.assert_array_equal(np.packbits(start.setup_m, axis=1), g["start_sm"])
    dev = DeviceInstance(inst)
    dev.set_variant(variant)
    sm, sr, trace, st = dev.vnd(start.setup_m, start.setup_r)
    assert st["cost"] == int(g["cost"]) == 4484593955
    np.testing.assert_array_equal(trace, g["trace"])
    np.testing.assert_array_equal(np.packbits(sm, axis=1), g["final_sm"])
    np.testing.assert_array_equal(np.packbits(sr, axis=1), g["final_sr"])
    assert st["evals_reference"] == int(g["evals"]) == 7814870
    assert st["moves"] == int(g["moves"]) and st["sweeps"] == int(g["sweeps"])


def _big():
    with open(os.path.join(GOLDEN, "big.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("variant", [8, 4, 64])
def test_c3_k100000_vnd_golden(variant):
    """BASELINE config 3 at full size: K=100,000, T=52 -- final cost
    449,100,704,810, full trace and plan hash from the live reference
    (warp-per-product kernel without / with the slack skip, and the
    lane-per-product kernel)."""
    g = _big()["k100000_t52"]
    inst = generate_instance(GeneratorConfig(products=100000, periods=52, seed=0))
    start = initial_solution(inst)
    assert _plan_sha(start.setup_m, start.setup_r) == g["start_plan_sha"]
    dev = DeviceInstance(inst)
    dev.set_variant(variant)
    sm, sr, trace, st = dev.vnd(start.setup_m, start.setup_r)
    assert st["cost"] == g["cost"] == 449100704810
    assert trace.tolist() == g["trace"]
    assert _plan_sha(sm, sr) == g["plan_sha"]


@pytest.mark.parametrize("variant", [0, 2])
def test_c4_t520_sample_golden(variant):
    """BASELINE config 4 (T=520): products of the K=10,000 seed-0 instance;
    per-product VND is exact by decomposition, so a sample pins the path."""
    g = _big()["k10000_t520_sample"]
    full = generate_instance(GeneratorConfig(products=10000, periods=520, seed=0))
    sub = g["products"]
    inst = Instance(len(sub), 520, full.demand[sub], full.returns[sub],
                    full.setup_cost_m[sub], full.setup_cost_r[sub], full.holding_cost_m[sub],
                    full.holding_cost_r[sub], full.unit_cost_m[sub], full.unit_cost_r[sub])
    start = initial_solution(inst)
    dev = DeviceInstance(inst)
    dev.set_variant(variant)   # 0: CTA per product (default), 2: warp per product
    sm, sr, trace, st = dev.vnd(start.setup_m, start.setup_r)
    assert st["cost"] == g["cost"]
    assert trace.tolist() == g["trace"]
    assert _plan_sha(sm, sr) == g["plan_sha"]


def _random_instance(rng, K, T, big=False):
    if big:   # force the int64 value / int64 cost paths
        dem = rng.integers(0, 10**8, size=(K, T))
        dem[rng.random((K, T)) < 0.3] = 0
        ret = (rng.random((K, T)) * dem * rng.uniform(0, 1)).astype(np.int64)
        c = [rng.integers(0, 10**9, size=K), rng.integers(0, 10**9, size=K),
             rng.integers(0, 1000, size=K), rng.integers(0, 1000, size=K),
             rng.integers(0, 1000, size=K), rng.integers(0, 1000, size=K)]
    else:
        dem = rng.integers(0, rng.integers(1, 120), size=(K, T))
        dem[rng.random((K, T)) < rng.uniform(0, 0.6)] = 0
        ret = (rng.random((K, T)) * dem * rng.uniform(0, 1.2)).astype(np.int64)
        c = [rng.integers(0, 300_000, size=K), rng.integers(0, 300_000, size=K),
             rng.integers(0, 600, size=K), rng.integers(0, 600, size=K),
             rng.integers(0, 50, size=K), rng.integers(0, 50, size=K)]
    return Instance(K, T, dem, ret, *c)


@pytest.mark.parametrize("variant", [8, 4, 2, 0, 64])
@pytest.mark.parametrize("seed", range(12))
def test_fuzz_against_oracle(seed, variant):
    rng = np.random.default_rng(1000 + seed)
    T = int(rng.choice([1, 2, 3, 5, 8, 31, 32, 33, 52, 63, 64, 65, 100, 150]))
    K = int(rng.integers(1, 60))
    big = seed % 4 == 3
    inst = _random_instance(rng, K, T, big)
    dev = DeviceInstance(inst)
    dev.set_variant(variant)
    plans = [initial_solution(inst)]
    plans.append(type(plans[0])(rng.random((K, T)) < 0.5, rng.random((K, T)) < 0.3))
    plans.append(type(plans[0])(np.ones((K, T), bool), rng.random((K, T)) < 0.5))
    for plan in plans:
        np.testing.assert_array_equal(dev.product_costs(plan.setup_m, plan.setup_r),
                                      oracle.product_costs(inst, plan.setup_m, plan.setup_r))
        for nbh in (1, 2, 3, 4):
            out, ev = dev.scan_products(plan.setup_m, plan.setup_r, nbh)
            want, oev = oracle.scan_products(inst, plan.setup_m, plan.setup_r, nbh)
            assert ev == oev
            np.testing.assert_array_equal(out[0], want[0])
            np.testing.assert_array_equal(out[1], want[1])
            np.testing.assert_array_equal(out[4], want[4])
            w = want[0] > 0
            for i in (2, 3):
                np.testing.assert_array_equal(out[i][w], want[i][w])
        for k_max in (2, 4):
            sm, sr, trace, st = dev.vnd(plan.setup_m, plan.setup_r, k_max)
            om, orr, ocost, otrace, ost = oracle.vnd(inst, plan.setup_m, plan.setup_r, k_max)
            assert st["cost"] == ocost
            np.testing.assert_array_equal(trace, otrace)
            np.testing.assert_array_equal(sm, om)
            np.testing.assert_array_equal(sr, orr)
            assert st["evals_reference"] == ost["evals"]


def test_wide_int64_path():
    """Values too large for int32 take the int64-value / int64-cost path."""
    rng = np.random.default_rng(77)
    K, T = 9, 40
    dem = rng.integers(10**8, 10**9, size=(K, T))
    dem[rng.random((K, T)) < 0.3] = 0
    ret = (rng.random((K, T)) * dem * 0.7).astype(np.int64)
    c = [rng.integers(0, 10**9, size=K), rng.integers(0, 10**9, size=K),
         rng.integers(0, 1000, size=K), rng.integers(0, 1000, size=K),
         rng.integers(0, 1000, size=K), rng.integers(0, 1000, size=K)]
    inst = Instance(K, T, dem, ret, *c)
    dev = DeviceInstance(inst)
    assert dev.info["value_bytes"] == 8 and dev.info["cost_bytes"] == 8
    start = initial_solution(inst)
    sm, sr, trace, st = dev.vnd(start.setup_m, start.setup_r)
    om, orr, ocost, otrace, ost = oracle.vnd(inst, start.setup_m, start.setup_r)
    assert st["cost"] == ocost
    np.testing.assert_array_equal(trace, otrace)
    np.testing.assert_array_equal(sm, om)
    np.testing.assert_array_equal(sr, orr)
    assert st["evals_reference"] == ost["evals"]


def test_out_of_range_instance_rejected():
    inst = Instance(1, 3, [[2**62, 0, 1]], [[0, 0, 0]], [1], [1], [1], [1])
    with pytest.raises(ValueError):
        DeviceInstance(inst)


@pytest.mark.parametrize("variant", [0, 2])
def test_mixed_width_t520_paths(variant):
    """T=520-style instances take the int32-value / int64-cost path."""
    inst = generate_instance(GeneratorConfig(products=6, periods=300, seed=3))
    dev = DeviceInstance(inst)
    dev.set_variant(variant)
    assert dev.info["value_bytes"] == 4 and dev.info["cost_bytes"] == 8
    start = initial_solution(inst)
    sm, sr, trace, st = dev.vnd(start.setup_m, start.setup_r)
    om, orr, ocost, otrace, _ = oracle.vnd(inst, start.setup_m, start.setup_r, threads=6)
    assert st["cost"] == ocost
    np.testing.assert_array_equal(trace, otrace)
    np.testing.assert_array_equal(sm, om)


@pytest.mark.parametrize("variant", [2, 130])
def test_t130_wide_costs_16bit_rows(variant):
    """The 16-bit-row kernel (T > 63, warp per product: variant bit 2) with
    costs beyond 32 bits: every third product here has setup costs x 10^3
    (costs ~2 x 10^10, cpre values far past 2^32); every result equals the
    oracle's, as on the 8-byte-row layout (variant 130)."""
    rng = np.random.default_rng(130)
    K, T = 36, 130
    inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=13))
    km, kr = inst.setup_cost_m.copy(), inst.setup_cost_r.copy()
    km[::3] *= 10**3
    kr[::3] *= 10**3
    inst = Instance(K, T, inst.demand, inst.returns, km, kr, inst.holding_cost_m,
                    inst.holding_cost_r, inst.unit_cost_m, inst.unit_cost_r)
    assert inst.demand.sum(1).max() < 2**16 and inst.returns.sum(1).max() < 2**16
    dev = DeviceInstance(inst)
    dev.set_variant(variant)
    assert dev.info["value_bytes"] == 4 and dev.info["cost_bytes"] == 8
    start = initial_solution(inst)
    s0 = oracle.product_costs(inst, start.setup_m, start.setup_r)
    assert (s0[::3] >= 2**32).all()
    plans = [start, type(start)(rng.random((K, T)) < 0.5, rng.random((K, T)) < 0.3)]
    for plan in plans:
        for k_max in (2, 4):
            sm, sr, trace, st = dev.vnd(plan.setup_m, plan.setup_r, k_max)
            om, orr, ocost, otrace, ost = oracle.vnd(inst, plan.setup_m, plan.setup_r, k_max,
                                                     threads=8)
            assert st["cost"] == ocost
            np.testing.assert_array_equal(trace, otrace)
            np.testing.assert_array_equal(sm, om)
            np.testing.assert_array_equal(sr, orr)
            assert st["evals_reference"] == ost["evals"]
    sm, sr, trace, st = dev.vnd_host(inst, start.setup_m, start.setup_r)
    om, orr, ocost, otrace, _ = oracle.vnd(inst, start.setup_m, start.setup_r, threads=8)
    assert st["cost"] == ocost
    np.testing.assert_array_equal(trace, otrace)
    np.testing.assert_array_equal(sm, om)


@pytest.mark.parametrize("over", [False, True])
@pytest.mark.parametrize("T", [52, 300])
def test_int32_coefficient_bound(T, over):
    """int32 values with int64 costs multiply in 32 x 32 -> 64 bits only
    while every coefficient (p_M + T h_M, p_R + p_M + T h_R, k_M, k_R) is
    below 2^30: at the bound the int32-value path is exact, one past it the
    instance takes the int64-value path (coef_bound, remlot_b200.cu)."""
    rng = np.random.default_rng(31 + T)
    K = 8
    dem = rng.integers(0, 101, size=(K, T))
    dem[rng.random((K, T)) < 0.2] = 0
    ret = (rng.random((K, T)) * dem * 0.5).astype(np.int64)
    lim = 2**30 - 1
    pm = rng.integers(0, 1000, size=K)
    pr = rng.integers(0, 1000, size=K)
    hm = (lim - pm) // T           # p_M + T h_M <= 2^30 - 1
    hr = (lim - pm - pr) // T      # p_R + p_M + T h_R <= 2^30 - 1
    km = np.full(K, lim)
    kr = rng.integers(lim // 2, lim, size=K)
    if over:
        km[3] = lim + 1
    inst = Instance(K, T, dem, ret, km, kr, hm, hr, pm, pr)
    dev = DeviceInstance(inst)
    assert dev.info["value_bytes"] == (8 if over else 4)
    assert dev.info["cost_bytes"] == 8
    start = initial_solution(inst)
    sm, sr, trace, st = dev.vnd(start.setup_m, start.setup_r)
    om, orr, ocost, otrace, ost = oracle.vnd(inst, start.setup_m, start.setup_r)
    assert st["cost"] == ocost
    np.testing.assert_array_equal(trace, otrace)
    np.testing.assert_array_equal(sm, om)
    np.testing.assert_array_equal(sr, orr)
    assert st["evals_reference"] == ost["evals"]
    np.testing.assert_array_equal(dev.product_costs(sm, sr),
                                  oracle.product_costs(inst, sm, sr))
    if over:
        # streamed into a handle laid out for int32 values: the per-chunk
        # check sees the coefficient and falls back to a full upload
        small = generate_instance(GeneratorConfig(products=K, periods=T, seed=1))
        dev2 = DeviceInstance(small)
        assert dev2.info["value_bytes"] == 4
        sm2, sr2, trace2, st2 = dev2.vnd_host(inst, start.setup_m, start.setup_r)
        assert st2["cost"] == ocost
        np.testing.assert_array_equal(trace2, otrace)
        np.testing.assert_array_equal(sm2, om)
        np.testing.assert_array_equal(sr2, orr)


def test_c3_vnd_host_pipelined_golden():
    """rl_vnd_host (chunked uploads overlapped with the descent, the bench's
    e2e call) reproduces the C3 golden, then serves a different instance of
    the same shape on the same handle exactly like a fresh handle does."""
    g = _big()["k100000_t52"]
    inst = generate_instance(GeneratorConfig(products=100000, periods=52, seed=0))
    other = generate_instance(GeneratorConfig(products=100000, periods=52, seed=5))
    start = initial_solution(inst)
    dev = DeviceInstance(other)   # handle holds a different instance
    sm, sr, trace, st = dev.vnd_host(inst, start.setup_m, start.setup_r)
    assert st["cost"] == g["cost"]
    assert trace.tolist() == g["trace"]
    assert _plan_sha(sm, sr) == g["plan_sha"]
    s2 = initial_solution(other)
    got = dev.vnd_host(other, s2.setup_m, s2.setup_r, k_max=3)
    want = DeviceInstance(other).vnd(s2.setup_m, s2.setup_r, k_max=3)
    assert got[3]["cost"] == want[3]["cost"]
    np.testing.assert_array_equal(got[2], want[2])
    np.testing.assert_array_equal(got[0], want[0])
    np.testing.assert_array_equal(got[1], want[1])
    assert got[3]["evals_reference"] == want[3]["evals_reference"]


def test_vnd_host_width_fallback():
    """New data wider than the handle's int32 layout fall back to a full
    upload (int64 path) with identical results; negative data are refused."""
    rng = np.random.default_rng(5)
    small = _random_instance(rng, 17, 40)
    wide = _random_instance(rng, 17, 40, big=True)
    dev = DeviceInstance(small)
    assert dev.info["value_bytes"] == 4
    start = initial_solution(wide)
    sm, sr, trace, st = dev.vnd_host(wide, start.setup_m, start.setup_r)
    om, orr, ocost, otrace, ost = oracle.vnd(wide, start.setup_m, start.setup_r)
    assert st["cost"] == ocost
    np.testing.assert_array_equal(trace, otrace)
    np.testing.assert_array_equal(sm, om)
    np.testing.assert_array_equal(sr, orr)
    # and back to small data on the (now int64) handle
    s0 = initial_solution(small)
    sm, sr, trace, st = dev.vnd_host(small, s0.setup_m, s0.setup_r)
    om, orr, ocost, otrace, _ = oracle.vnd(small, s0.setup_m, s0.setup_r)
    assert st["cost"] == ocost
    np.testing.assert_array_equal(trace, otrace)
    bad = Instance(17, 40, -np.ones((17, 40), np.int64), small.returns, *small.arrays()[2:])
    with pytest.raises(ValueError):
        dev.vnd_host(bad, s0.setup_m, s0.setup_r)


def test_product_stats_and_variant_guard():
    """rl_vnd_product_stats: per-product sweeps/moves/evals of the last
    descent add up to the totals (global sweeps = the slowest product's);
    the removed two-products-per-warp variant bit is rejected."""
    inst = generate_instance(GeneratorConfig(products=300, periods=52, seed=0))
    start = initial_solution(inst)
    dev = DeviceInstance(inst)
    with pytest.raises(Exception):
        dev.set_variant(1)
    _, _, trace, st = dev.vnd(start.setup_m, start.setup_r)
    sw, mv, ev = dev.product_stats()
    assert int(sw.max()) == st["sweeps"] == (len(trace) - 1) // 4
    assert int(mv.sum()) == st["moves"]
    assert int(ev.sum()) == st["evals"]
    assert st["cost"] == 1328299635   # live-reference golden


@pytest.mark.parametrize("K,T", [(6, 3000), (2, 7000)])
def test_long_horizon_shared_memory_limits(K, T):
    """Horizons whose per-product shared memory does not fit four slots per
    CTA (T=3000: ~79 KB per product) run with fewer warps per CTA; T=7000
    (~184 KB) fits one product per CTA.  Single passes match the oracle, and
    the descent ends in a local optimum of N1..N4 whose cost is the plan's
    cost, identically for the CTA-per-product and warp-per-product kernels."""
    rng = np.random.default_rng(T)
    inst = _random_instance(rng, K, T)
    start = initial_solution(inst)
    dev = DeviceInstance(inst)
    np.testing.assert_array_equal(dev.product_costs(start.setup_m, start.setup_r),
                                  oracle.product_costs(inst, start.setup_m, start.setup_r))
    for nbh in (1, 3):
        out, ev = dev.scan_products(start.setup_m, start.setup_r, nbh)
        want, oev = oracle.scan_products(inst, start.setup_m, start.setup_r, nbh)
        assert ev == oev
        np.testing.assert_array_equal(out[0], want[0])
    results = []
    for variant in (0, 2):
        dev.set_variant(variant)
        sm, sr, trace, st = dev.vnd(start.setup_m, start.setup_r)
        results.append((sm.tobytes(), sr.tobytes(), trace.tolist(), st["cost"]))
        assert st["cost"] == trace[-1] == int(dev.product_costs(sm, sr).sum())
        for nbh in (1, 2, 3, 4):
            out, _ = dev.scan_products(sm, sr, nbh)
            assert not out[0].any()
    assert results[0] == results[1]
