"""Exhaustive optimum on the GPU (mirror of the reference module oracle.py;
named exhaustive.py here so it is not confused with the CPU test oracle/).

Products are independent, so the optimum factorizes per product; every one
of the 2^(2T) setup patterns is decoded with the search's own policy
(reference oracle.py:1-44, _kernels.oracle_product :347-371), one GPU thread
per pattern.  Tractable only for short horizons (T <= 10, like the
reference).  SURVEY.md 8(f) row 2.
"""

from . import _native
from .model import Instance
from .plan import SetupPlan

MAX_PERIODS = 10


def enumerate_optimal(inst: Instance):
    """(cost, plan) minimising the decoded cost per product (oracle.py:19-44)."""
    T = inst.periods
    if T > MAX_PERIODS:
        raise ValueError(f"exhaustive enumeration needs periods <= {MAX_PERIODS} "
                         f"(2^(2*{T}) patterns per product is intractable)")
    costs, sm, sr = _native.device_instance(inst).oracle_optimal()
    return int(costs.sum()), SetupPlan(sm, sr)
