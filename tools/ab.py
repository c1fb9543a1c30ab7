"""A/B kernel variants (rl_instance_set_variant bits) on BASELINE workloads.

    python tools/ab.py c3 0,4,8 [reps]

Prints the best-of-reps VND kernel time and the final cost per variant.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig, generate_instance  # noqa: E402
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

SIZES = {"c3": (100000, 52), "c2": (1000, 52), "c4": (10000, 520), "c4s": (100, 520),
         "t30": (20000, 30), "t63": (20000, 63), "t64": (20000, 64), "t100": (20000, 100), "t200": (10000, 200), "t130": (15000, 130), "k100": (100, 52), "k500": (500, 52)}
names = sys.argv[1].split(",")
variants = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
for name in names:
    K, T = SIZES[name]
    inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=0))
    dev = DeviceInstance(inst)
    sm, sr = dev.initial_solution()
    for v in variants:
        dev.set_variant(v)
        dev.vnd(sm, sr)
        best = None
        for _ in range(reps):
            _, _, tr, st = dev.vnd(sm, sr)
            ms = st["kernel_ns"] / 1e6
            best = ms if best is None else min(best, ms)
        print(f"{name} K={K} T={T} variant {v}: {best:.3f} ms cost {st['cost']} "
              f"evals {st['evals']} ref {st['evals_reference']} trace {len(tr)}", flush=True)
