"""Speculative GVNS batches: rounds consumed per batch and batch latency.

    python tools/gvns_batch_probe.py W R b1,b2,...
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig, generate_instance, initial_solution  # noqa
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

W, R = int(sys.argv[1]), int(sys.argv[2])
inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
init = initial_solution(inst)
dev = DeviceInstance(inst)
for B in [int(b) for b in sys.argv[3].split(",")]:
    for rep in range(2):
        dev.gvns_begin(W, 5, 4, 0, init.setup_m, init.setup_r, batch=B)
        calls, fb = 0, 0
        t0 = time.perf_counter()
        rounds = 0
        while rounds < R:
            dev.gvns_run(R)
            calls += 1
            _, _, info = dev.gvns_state(0, want_plan=False)
            rounds = info["rounds"]
            fb += info["fallbacks"]
        dt = time.perf_counter() - t0
    print(f"W={W} B={B}: {R} rounds in {calls} batches ({R / calls:.1f} rounds/batch), "
          f"{dt / calls * 1e6:.0f} us/batch, {R / dt:.0f} rounds/s, accepted {info['accepted']}, "
          f"fallbacks {fb}, cost {info['inc_cost']}", flush=True)
