"""Two end-to-end descents through rl_vnd_host (host buffers, chunked
uploads overlapped with the descent) at C3, for ncu launch lists of the
instance-streaming kernels (k_check_narrow) beside k_vnd."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig  # noqa: E402
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

dev = DeviceInstance.generate(GeneratorConfig(products=100000, periods=52, seed=0))
inst = dev.download()
sm, sr = dev.initial_solution()
for _ in range(2):
    _, _, _, st = dev.vnd_host(inst, sm, sr)
print(st)
