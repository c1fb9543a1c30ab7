"""One warm + one profiled VND of a BASELINE workload (for ncu captures).

    python tools/profile_vnd.py [c3|c2|c4]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig, generate_instance  # noqa: E402
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

SIZES = {"c3": (100000, 52), "c2": (1000, 52), "c4": (10000, 520)}
K, T = SIZES[sys.argv[1] if len(sys.argv) > 1 else "c3"]
inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=0))
dev = DeviceInstance(inst)
sm, sr = dev.initial_solution()
for _ in range(2):
    _, _, _, st = dev.vnd(sm, sr)
print(K, T, st)
