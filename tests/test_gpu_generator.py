"""rl_generate_instance (device generator) vs model.generate_instance, whose
draws are pinned to the live reference (tests/test_model.py); bit-exact."""

import numpy as np
import pytest

from paper_1704_05132_b200 import GeneratorConfig, generate_instance, initial_solution
from paper_1704_05132_b200._native import DeviceInstance

pytestmark = pytest.mark.gpu

CONFIGS = [
    dict(products=1000, periods=52, seed=0),                  # C2
    dict(products=300, periods=1, seed=7, demand_max=3),      # many all-zero rows redrawn
    dict(products=40, periods=7, seed=2**40 + 3, demand_max=1, return_ratio=1.0),
    dict(products=20, periods=13, seed=123, demand_max=0, return_ratio=0.3),
    dict(products=100, periods=20, seed=5, demand_max=4_000_000_000, return_ratio=0.9),
    dict(products=64, periods=33, seed=2**64 - 1, setup_cost_range=(0, 2**32 - 2),
         holding_cost_range=(7, 7), unit_cost_range=(3, 900)),
    dict(products=10, periods=520, seed=11, return_ratio=0.0),
]


def _same(a, b):
    assert a.products == b.products and a.periods == b.periods
    for x, y in zip(a.arrays(), b.arrays()):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: f"K{c['products']}T{c['periods']}")
def test_generate_matches_host(cfg):
    config = GeneratorConfig(**cfg)
    _same(DeviceInstance.generate(config).download(), generate_instance(config))


def test_generate_shard_slices():
    config = GeneratorConfig(products=5000, periods=52, seed=3)
    host = generate_instance(config)
    for lo, hi in [(0, 1250), (1250, 2500), (4999, 5000)]:
        _same(DeviceInstance.generate(config, lo, hi).download(), host.slice(lo, hi))


def test_generate_c3_and_descend():
    """The C3 instance generated on the device descends to the golden cost."""
    config = GeneratorConfig(products=100000, periods=52, seed=0)
    dev = DeviceInstance.generate(config)
    inst = dev.download()
    _same(inst, generate_instance(config))
    start = initial_solution(inst)
    sm, sr, trace, st = dev.vnd(start.setup_m, start.setup_r)
    assert st["cost"] == 449100704810


def test_generate_rejects_bad_config():
    with pytest.raises(ValueError):
        DeviceInstance.generate(GeneratorConfig(products=5, periods=5, demand_max=2**33))
    with pytest.raises(ValueError):
        DeviceInstance.generate(GeneratorConfig(products=5, periods=5), 3, 3)
