"""Small workload touching every kernel, for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1704_05132_b200 import (GeneratorConfig, SetupPlan, SolverConfig, decode,  # noqa: E402
                                   enumerate_optimal, evaluate, generate_instance, gvns,
                                   initial_solution, vnd, vnd_pass, enumerate_neighbors)
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402

for K, T in ((40, 52), (6, 130), (3, 5)):
    inst = generate_instance(GeneratorConfig(products=K, periods=T, seed=1))
    start = initial_solution(inst)
    for variant in (0, 2, 4, 8, 16, 64, 128, 256):
        dev = DeviceInstance(inst)
        dev.set_variant(variant)
        dev.vnd(start.setup_m, start.setup_r)
    plan, cost = vnd(inst, start)
    for nbh in (1, 2, 3, 4):
        vnd_pass(inst, plan, nbh)
        enumerate_neighbors(plan, nbh, 0)
    decode(inst, plan)
    evaluate(inst, SetupPlan(np.ones((K, T), bool), np.zeros((K, T), bool)))
    gvns(inst, SolverConfig(t_max=1e9, workers=3, seed=2, max_rounds=4))
    if T <= 10:
        enumerate_optimal(inst)
print("sanitize workload done")
