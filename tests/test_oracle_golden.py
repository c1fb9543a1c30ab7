"""Pins the CPU oracle (oracle/) to fixtures made by the live reference.

The oracle is the checker for the CUDA path, so it must itself agree with
the reference bit-for-bit on every golden vector before it is trusted
(tests/golden/gen_golden.py made the fixtures by importing remlot)."""

import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, GoldInstance, golden

NAMES = ("dec", "p0", "m0", "r0", "p1", "m1", "r1")


def _cases(small_cases):
    for idx, K, T in small_cases["cases"]:
        inst = GoldInstance(small_cases, f"c{idx}_")
        for pi in range(int(small_cases["n_plans"])):
            yield inst, f"c{idx}_{pi}_"


def test_row_costs_match_reference(small_cases):
    n = 0
    for inst, p in _cases(small_cases):
        got = oracle.product_costs(inst, small_cases[p + "sm"], small_cases[p + "sr"])
        np.testing.assert_array_equal(got, small_cases[p + "cost"])
        n += 1
    assert n >= 150


def test_list_moves_match_reference(small_cases):
    for inst, p in _cases(small_cases):
        sm, sr = small_cases[p + "sm"], small_cases[p + "sr"]
        for nbh in (1, 2, 3, 4):
            ns = small_cases[p + f"lm{nbh}_n"]
            for k in range(inst.products):
                got = oracle.list_moves(nbh, sm[k], sr[k])
                n = int(ns[k])
                assert len(got[0]) == n
                for name, g in zip(("mp0", "mm0", "mr0", "mp1", "mm1", "mr1"), got):
                    np.testing.assert_array_equal(g, small_cases[p + f"lm{nbh}_{name}"][k, :n])


def test_scan_products_match_reference(small_cases):
    for inst, p in _cases(small_cases):
        for nbh in (1, 2, 3, 4):
            out, _ = oracle.scan_products(inst, small_cases[p + "sm"], small_cases[p + "sr"], nbh)
            for name, g in zip(NAMES, out):
                np.testing.assert_array_equal(g, small_cases[p + f"scan{nbh}_{name}"],
                                              err_msg=f"{p} nbh={nbh} {name}")


@pytest.mark.parametrize("threads", [1, 3])
def test_vnd_matches_reference(small_cases, threads):
    for inst, p in _cases(small_cases):
        for k_max in (1, 4):
            sm, sr, cost, trace, _ = oracle.vnd(inst, small_cases[p + "sm"],
                                                small_cases[p + "sr"], k_max, threads)
            assert cost == int(small_cases[p + f"vnd{k_max}_cost"])
            np.testing.assert_array_equal(trace, small_cases[p + f"vnd{k_max}_trace"])
            np.testing.assert_array_equal(sm, small_cases[p + f"vnd{k_max}_sm"])
            np.testing.assert_array_equal(sr, small_cases[p + f"vnd{k_max}_sr"])


def test_initial_solution_matches_reference(small_cases):
    for inst, p in _cases(small_cases):
        if not p.endswith("_0_"):
            continue
        sm, sr = oracle.initial_solution(inst)
        np.testing.assert_array_equal(sm, small_cases[p + "sm"])
        np.testing.assert_array_equal(sr, small_cases[p + "sr"])


def test_c1_trajectory_every_pass():
    """K=10 T=52 seed 0 (BASELINE config 1): every lockstep pass's scan
    outputs, the 181-entry trace and the final cost 44,066,661."""
    from paper_1704_05132_b200.model import GeneratorConfig, generate_instance
    g = golden("c1_trajectory.npz")
    inst = generate_instance(GeneratorConfig(products=10, periods=52, seed=0))
    sm, sr = g["start_sm"].copy(), g["start_sr"].copy()
    np.testing.assert_array_equal(np.stack(oracle.initial_solution(inst)), np.stack([sm, sr]))
    for i in range(g["pass_dec"].shape[0]):
        nbh = i % 4 + 1
        out, _ = oracle.scan_products(inst, sm, sr, nbh)
        for name, got in zip(NAMES, out):
            np.testing.assert_array_equal(got, g["pass_" + name][i], err_msg=f"pass {i} {name}")
        sm8, sr8 = sm.astype(np.uint8), sr.astype(np.uint8)
        oracle.lib().orc_apply_scan(52, 0, 10, *[oracle._ptr(np.ascontiguousarray(
            a, dtype=np.int64 if a.dtype != bool else np.uint8)) for a in out],
            oracle._ptr(sm8), oracle._ptr(sr8))
        sm, sr = sm8.astype(bool), sr8.astype(bool)
    np.testing.assert_array_equal(sm, g["final_sm"])
    fm, fr, cost, trace, stats = oracle.vnd(inst, g["start_sm"], g["start_sr"])
    assert cost == int(g["cost"]) == 44066661
    np.testing.assert_array_equal(trace, g["trace"])
    assert stats == dict(evals=int(g["evals"]), moves=int(g["moves"]), sweeps=int(g["sweeps"]))


def test_k1000_vnd_golden():
    from paper_1704_05132_b200.model import GeneratorConfig, generate_instance
    g = golden("k1000.npz")
    inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
    sm0, sr0 = oracle.initial_solution(inst)
    np.testing.assert_array_equal(np.packbits(sm0, axis=1), g["start_sm"])
    sm, sr, cost, trace, stats = oracle.vnd(inst, sm0, sr0, threads=8)
    assert cost == int(g["cost"]) == 4484593955
    np.testing.assert_array_equal(trace, g["trace"])
    np.testing.assert_array_equal(np.packbits(sm, axis=1), g["final_sm"])
    np.testing.assert_array_equal(np.packbits(sr, axis=1), g["final_sr"])
    assert stats["evals"] == int(g["evals"]) == 7814870
    assert stats["sweeps"] == int(g["sweeps"])
