"""Host (numpy) vs device generate_instance wall time.  Usage: gen_time.py K T"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig, generate_instance  # noqa: E402
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
T = int(sys.argv[2]) if len(sys.argv) > 2 else 52
cfg = GeneratorConfig(products=K, periods=T, seed=0)
DeviceInstance.generate(GeneratorConfig(products=1000, periods=T, seed=1))   # warm
for rep in range(2):
    t0 = time.perf_counter()
    dev = DeviceInstance.generate(cfg)
    t1 = time.perf_counter()
    host = generate_instance(cfg)
    t2 = time.perf_counter()
    print(f"K={K} T={T}: device generate+prepare {1e3 * (t1 - t0):.1f} ms, "
          f"host numpy {1e3 * (t2 - t1):.1f} ms", flush=True)
    del dev
