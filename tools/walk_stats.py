"""Delta-walk statistics of one descent (diagnostic build, -DRL_WALK_STATS).

    tools/walk_stats.sh   (builds libremlot_b200_walkstats.so, runs this)

Per neighborhood pass: loop iterations of the lane work queue, moves, walk
steps, the longest walk and the busiest lane.  Lane utilisation of the walk
loop = steps / (32 x iterations); a pass whose iterations equal its longest
walk is bound by that walk, not by the number of moves.
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig, generate_instance  # noqa: E402
from paper_1704_05132_b200 import _native  # noqa: E402
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

SIZES = {"c3": (100000, 52), "c2": (1000, 52), "c4": (10000, 520)}
lib = _native.load()
lib.rl_walk_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(160, np.int64)
variants = [int(v) for v in os.environ.get("RL_VARIANTS", "0").split(",")]
for name, variant in [(n, v) for n in (sys.argv[1:] or ["c2", "c3"]) for v in variants]:
    K, T = SIZES[name]
    inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=0))
    dev = DeviceInstance(inst)
    dev.set_variant(variant)
    sm, sr = dev.initial_solution()
    lib.rl_walk_stats(_native.ptr(buf), 1)
    _, _, _, st = dev.vnd(sm, sr)
    lib.rl_walk_stats(_native.ptr(buf), 1)
    P, it, n, steps, mx, busy = (int(x) for x in buf[:6])
    print(f"{name} K={K} T={T} variant {variant}: passes {P}, moves/pass {n / P:.1f}, steps/move {steps / n:.2f}, "
          f"iterations/pass {it / P:.2f}, longest walk/pass {mx / P:.2f}, busiest lane/pass "
          f"{busy / P:.2f}, lane utilisation {steps / (32 * it):.3f}, set-up branches/pass "
          f"{int(buf[6]) / P:.2f}")
    h = buf[8:72]
    print("  walk-length histogram (len:count%): " +
          " ".join(f"{i}:{100 * h[i] / h.sum():.1f}" for i in range(64) if h[i] * 1000 > h.sum()))
    print("  per neighborhood (passes, improving fraction, moves/pass): " + "  ".join(
        f"N{j}: {buf[136 + j]} {buf[144 + j] / max(buf[136 + j], 1):.3f} "
        f"{buf[152 + j] / max(buf[136 + j], 1):.1f}" for j in range(1, 5)))
    h = buf[72:136]
    print("  iterations/pass histogram: " +
          " ".join(f"{i}:{100 * h[i] / h.sum():.1f}" for i in range(64) if h[i] * 1000 > h.sum()))
