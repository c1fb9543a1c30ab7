"""Lane-state statistics of the lane-per-product VND (diagnostic build).

    tools/walk_stats.sh builds libremlot_b200_walkstats.so;
    REMLOT_B200_LIB=<that> python tools/lane_stats.py c3
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig  # noqa: E402
from paper_1704_05132_b200 import _native  # noqa: E402
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

SIZES = {"c3": (100000, 52), "c2": (1000, 52), "k200k": (200000, 52)}
lib = _native.load()
lib.rl_lane_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(16, np.int64)
for name in sys.argv[1:] or ["c3"]:
    K, T = SIZES[name]
    dev = DeviceInstance.generate(GeneratorConfig(products=K, periods=T, seed=0))
    dev.set_variant(64)
    sm, sr = dev.initial_solution()
    lib.rl_lane_stats(_native.ptr(buf), 1)
    _, _, _, st = dev.vnd(sm, sr)
    lib.rl_lane_stats(_native.ptr(buf), 1)
    it = buf[0]
    print(f"{name}: kernel {st['kernel_ns'] / 1e6:.2f} ms, warp iterations {it}, per iteration: "
          f"walking {buf[1] / it:.2f}, idle {buf[2] / it:.2f}, done {buf[3] / it:.2f} lanes; "
          f"control steps {buf[4] / it:.3f}/iter with {buf[5] / max(buf[4], 1):.2f} lanes; "
          f"products {buf[6]}, load {buf[7] / max(buf[6], 1):.0f} cyc/product, "
          f"warp lifetime {buf[9] / max(1, it) * it:.3e} cyc total, "
          f"cycles/iteration {buf[9] / it:.1f}")
