"""Tail probe of the warp-per-product kernel (k_vnd, the default variant):
kernel time on the generator order, on products sorted by their measured
work (heaviest first: the LPT bound of the dynamic product queue), and on a
random order.  The gap between the first two is the share of the launch the
last products' tail costs.

    python tools/tail_probe.py c4     # K=10,000 T=520
    python tools/tail_probe.py c3     # K=100,000 T=52
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig  # noqa: E402
from paper_1704_05132_b200.model import Instance, COST_FIELDS  # noqa: E402
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

K, T = {"c3": (100000, 52), "c4": (10000, 520)}[sys.argv[1] if len(sys.argv) > 1 else "c4"]
dev = DeviceInstance.generate(GeneratorConfig(products=K, periods=T, seed=0))
inst = dev.download()
sm, sr = dev.initial_solution()
dev.vnd(sm, sr)
_, _, ev = dev.product_stats()
print(f"K={K} T={T}: evals per product mean {ev.mean():.0f} max {ev.max()} "
      f"(max/mean {ev.max() / ev.mean():.1f})", flush=True)


def timed(perm, label):
    sub = Instance(K, T, inst.demand[perm], inst.returns[perm],
                   *(getattr(inst, f)[perm] for f in COST_FIELDS))
    d = DeviceInstance(sub)
    a, b = d.initial_solution()
    d.vnd(a, b)
    ms = []
    for _ in range(3):
        _, _, _, st = d.vnd(a, b)
        ms.append(st["kernel_ns"] / 1e6)
    print(f"{label}: {min(ms):.2f} ms cost {st['cost']}", flush=True)


timed(np.arange(K), "generator order")
timed(np.argsort(-ev, kind="stable"), "heaviest first (LPT bound)")
timed(np.random.default_rng(0).permutation(K), "random order")
