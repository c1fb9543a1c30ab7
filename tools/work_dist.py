"""Work distribution over products and the single-product latency floor.

    python tools/work_dist.py [c3|c4|c2]

Prints the per-product sweep/evaluation distribution of the descent, then
times sub-instances made of the heaviest products (1, one per SM, ...) and
prefixes of the instance: if the kernel time of the full workload is close
to the heaviest product's solo time, the launch is tail-bound, not
throughput-bound.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig, generate_instance  # noqa: E402
from paper_1704_05132_b200.model import Instance  # noqa: E402
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

SIZES = {"c3": (100000, 52), "c2": (1000, 52), "c4": (10000, 520)}
K, T = SIZES[sys.argv[1] if len(sys.argv) > 1 else "c4"]
inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=0))


def take(inst, idx):
    a = inst.arrays()
    return Instance(len(idx), inst.periods, a[0][idx], a[1][idx], *[x[idx] for x in a[2:]])


def kernel_ms(sub, reps=2, variant=None):
    dev = DeviceInstance(sub)
    if variant is not None:
        dev.set_variant(variant)
    sm, sr = dev.initial_solution()
    best = None
    for _ in range(reps):
        _, _, _, st = dev.vnd(sm, sr)
        ms = st["kernel_ns"] / 1e6
        best = ms if best is None else min(best, ms)
    return best, dev, st


ms, dev, st = kernel_ms(inst)
sw, mv, ev = dev.product_stats()
print(f"K={K} T={T}: kernel {ms:.2f} ms, global sweeps {st['sweeps']}, evals {st['evals']}")
for name, a in (("sweeps", sw), ("moves", mv), ("evals", ev)):
    q = np.percentile(a, [50, 90, 99, 99.9, 100])
    print(f"  {name:6s} mean {a.mean():10.1f}  p50/p90/p99/p99.9/max " +
          " ".join(f"{x:.0f}" for x in q))
order = np.argsort(-ev, kind="stable")
print(f"  heaviest product {order[0]}: {ev[order[0]]} evals, {sw[order[0]]} sweeps; "
      f"mean evals x (K / resident warps) bound")
for n in (1, 148, 592):
    if n > K:
        continue
    sub = take(inst, order[:n])
    for variant in ((None, 2) if T > 63 else (None,)):
        m, _, _ = kernel_ms(sub, variant=variant)
        print(f"  heaviest {n:5d} products (variant {variant}): {m:.2f} ms", flush=True)
for frac in (0.25, 0.5):
    n = int(K * frac)
    m, _, _ = kernel_ms(inst.slice(0, n))
    print(f"  first {n} products: {m:.2f} ms", flush=True)
