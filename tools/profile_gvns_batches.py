"""Device GVNS through the per-batch API (rl_gvns_run, plain CUDA-graph
replays) instead of the conditional-node loop, so that ncu sees every
kernel launch.  python tools/profile_gvns_batches.py [workers] [rounds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1704_05132_b200 import GeneratorConfig, generate_instance, initial_solution  # noqa
from paper_1704_05132_b200._native import DeviceInstance  # noqa: E402
from paper_1704_05132_b200.gvns import _batch  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
R = int(sys.argv[2]) if len(sys.argv) > 2 else 200
inst = generate_instance(GeneratorConfig(products=1000, periods=52, seed=0))
dev = DeviceInstance(inst)
init = initial_solution(inst)
dev.gvns_begin(W, 5, 4, 0, init.setup_m, init.setup_r, batch=_batch(W))
rounds = 0
while rounds < R:
    dev.gvns_run(R)
    rounds = dev.gvns_state(0, want_plan=False)[2]["rounds"]
print("rounds", rounds, "cost", dev.gvns_state(0, want_plan=False)[2]["inc_cost"])
