import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


class GoldInstance:
    """Instance-shaped view of fixture arrays (used with the oracle)."""

    def __init__(self, data, prefix):
        self.demand = data[prefix + "demand"]
        self.returns = data[prefix + "returns"]
        self.products, self.periods = self.demand.shape
        for f in ("setup_cost_m", "setup_cost_r", "holding_cost_m",
                  "holding_cost_r", "unit_cost_m", "unit_cost_r"):
            setattr(self, f, data[prefix + f])


@pytest.fixture(scope="session")
def small_cases():
    return golden("small_cases.npz")
