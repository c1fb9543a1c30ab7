"""Compare the e2e leg: rl_vnd_host (pipelined) vs rl_instance_update + rl_vnd.
Usage: python tools/e2e_compare.py [K] [T] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1704_05132_b200 import GeneratorConfig, _native, devbench, generate_instance  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
T = int(sys.argv[2]) if len(sys.argv) > 2 else 52
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=0))
dev = _native.DeviceInstance(inst)
for rep in range(2):
    for pipe in (False, True):
        ms, h2d, d2h = devbench.e2e_steps(torch, _native, dev, inst, steps, 1, None, "cpu",
                                          pipelined=pipe)
        print(f"K={K} T={T} pipelined={pipe}: {ms / steps:.3f} ms/step "
              f"(h2d {h2d / 1e6:.1f} MB, d2h {d2h / 1e6:.1f} MB)", flush=True)
