"""Tail probe of the lane-per-product kernel at C3: kernel time on the
generator order, on products sorted by their measured work (heaviest first:
the LPT bound), and on a random order."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig  # noqa: E402
from paper_1704_05132_b200.model import Instance, COST_FIELDS  # noqa: E402
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

K, T = 100000, 52
dev = DeviceInstance.generate(GeneratorConfig(products=K, periods=T, seed=0))
inst = dev.download()
sm, sr = dev.initial_solution()
dev.set_variant(32)
dev.vnd(sm, sr)
_, _, ev = dev.product_stats()


def timed(perm, label):
    sub = Instance(K, T, inst.demand[perm], inst.returns[perm],
                   *(getattr(inst, f)[perm] for f in COST_FIELDS))
    d = DeviceInstance(sub)
    d.set_variant(64)
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
timed(np.argsort(ev, kind="stable"), "lightest first")
