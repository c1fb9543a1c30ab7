"""A few device GVNS rounds (for ncu launch lists / timing).

    python tools/profile_gvns.py [workers] [rounds]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig, SolverConfig, generate_instance, gvns  # noqa

W = int(sys.argv[1]) if len(sys.argv) > 1 else 128
R = int(sys.argv[2]) if len(sys.argv) > 2 else 20
inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
if os.environ.get("RL_VARIANT"):   # A/B of kernel variant bits on the cached handle
    from paper_1704_05132_b200._native import device_instance
    device_instance(inst).set_variant(int(os.environ["RL_VARIANT"]))
gvns(inst, SolverConfig(t_max=1e9, workers=W, seed=0, max_rounds=2))
t0 = time.perf_counter()
res = gvns(inst, SolverConfig(t_max=1e9, workers=W, seed=0, max_rounds=R))
dt = time.perf_counter() - t0
print(f"W={W} rounds={res.rounds} {dt * 1e3:.1f} ms ({res.rounds / dt:.0f} rounds/s) cost {res.cost}")
