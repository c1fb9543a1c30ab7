"""Dev timing: VND kernel time for C2/C3/C4 (both k_vnd variants for T<=64)."""
import sys
import time

sys.path.insert(0, '.')  # run from the repo root
from paper_1704_05132_b200 import GeneratorConfig, generate_instance  # noqa: E402
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

for K, T in ((1000, 52), (100000, 52), (10000, 520)):
    inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=0))
    dev = DeviceInstance(inst)
    sm, sr = dev.initial_solution()
    for packed in ((1, 0) if T <= 63 else (0, 2)):
        dev.set_variant(packed)
        for rep in range(3):
            t0 = time.perf_counter()
            m, r, tr, st = dev.vnd(sm, sr)
            t1 = time.perf_counter()
            print(f"K={K} T={T} packed={packed} wall {1e3 * (t1 - t0):.1f} ms "
                  f"kernel {st['kernel_ns'] / 1e6:.2f} ms cost {st['cost']} scored {st.get('evals_scored')} "
                  f"of {st['evals']}", flush=True)

# latency-bound long horizon: few products
inst = generate_instance(GeneratorConfig(products=100, periods=520, seed=0))
dev = DeviceInstance(inst)
sm, sr = dev.initial_solution()
for packed in (0, 2):
    dev.set_variant(packed)
    m, r, tr, st = dev.vnd(sm, sr)
    m, r, tr, st = dev.vnd(sm, sr)
    print(f"K=100 T=520 variant={packed} kernel {st['kernel_ns'] / 1e6:.2f} ms cost {st['cost']}")
