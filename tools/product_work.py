"""Per-product VND work at a workload (sweeps, moves, performed evaluations)
dumped to gpurun_out/product_work_<wl>.npz for scheduling analysis."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig  # noqa: E402
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

SIZES = {"c3": (100000, 52), "c4": (10000, 520)}
wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
K, T = SIZES[wl]
dev = DeviceInstance.generate(GeneratorConfig(products=K, periods=T, seed=0))
dev.set_variant(32)
sm, sr = dev.initial_solution()
dev.vnd(sm, sr)
sw, mv, ev = dev.product_stats()
np.savez_compressed(f"gpurun_out/product_work_{wl}.npz", sweeps=sw, moves=mv, evals=ev)
print(wl, "evals mean", ev.mean(), "max", ev.max(), "sweeps max", sw.max())
