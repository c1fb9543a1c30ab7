"""A/B of kernel variants on one workload: kernel ms (CUDA events of the
descent, best of 5) and the cost check.

    python tools/ab_vnd.py c3 0 32 ...   (variant bits, see _native.set_variant)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig  # noqa: E402
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

SIZES = {"c3": (100000, 52), "c2": (1000, 52), "c4": (10000, 520), "t63": (50000, 63),
         "t30": (100000, 30), "k20k": (20000, 52), "k50k": (50000, 52), "k200k": (200000, 52),
         "k12k": (12500, 52), "k25k": (25000, 52), "t200": (20000, 200), "k100t520": (100, 520), "k296t520": (296, 520)}
wl = sys.argv[1]
K, T = SIZES[wl]
dev = DeviceInstance.generate(GeneratorConfig(products=K, periods=T, seed=0))
sm, sr = dev.initial_solution()
for v in [int(x) for x in sys.argv[2:]]:
    dev.set_variant(v)
    dev.vnd(sm, sr)
    ms = []
    for _ in range(5):
        _, _, tr, st = dev.vnd(sm, sr)
        ms.append(st["kernel_ns"] / 1e6)
    print(f"{wl} K={K} T={T} variant={v}: best {min(ms):.3f} ms  median {sorted(ms)[2]:.3f} ms  "
          f"cost {st['cost']} sweeps {st['sweeps']} evals_ref {st['evals_reference']}",
          flush=True)
