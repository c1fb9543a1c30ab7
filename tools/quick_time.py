import time, sys
sys.path.insert(0, '.')
import numpy as np
from paper_1704_05132_b200 import GeneratorConfig, generate_instance, initial_solution
from paper_1704_05132_b200._native import DeviceInstance
for K, T in ((1000, 52), (100000, 52), (10000, 520)):
    inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=0))
    dev = DeviceInstance(inst)
    sm, sr = dev.initial_solution()
    for rep in range(3):
        t0 = time.perf_counter()
        m, r, tr, st = dev.vnd(sm, sr)
        t1 = time.perf_counter()
        print(K, T, dev.info, f"wall {1e3*(t1-t0):.1f} ms kernel {st['kernel_ns']/1e6:.2f} ms", st, flush=True)
