import sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_1704_05132_b200 import GeneratorConfig, generate_instance
from paper_1704_05132_b200._native import DeviceInstance
cfg = GeneratorConfig(products=800000, periods=52, seed=0)
t0 = time.perf_counter()
dev = DeviceInstance.generate(cfg, 700000, 800000)
sub = dev.download()
t1 = time.perf_counter()
host = generate_instance(cfg).slice(700000, 800000)
t2 = time.perf_counter()
ok = all(np.array_equal(a, b) for a, b in zip(sub.arrays(), host.arrays()))
print(f"shard 7/8 of K=800k: device {1e3*(t1-t0):.0f} ms, host {1e3*(t2-t1):.0f} ms, identical={ok}")
