"""Paper-scale quality at equal wall time (the reference's
full-scale experiment of bench.py:145-154: 300 products x 52 periods, the four
schemes of gvns.py:22-27, 60 s per cell, solver seed 1).

    # in the build container, the live reference (numba, 8 host cores):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tools/paper_scale.py cpu [n_instances] [t_max]
    # on a B200 (the drop-in):
    python tools/paper_scale.py gpu [n_instances] [t_max]

cpu writes tests/golden/paper_scale_cpu.json (objective, rounds, wall per
cell).  gpu runs the same cells on the device with the same budget, and --
because GVNS is deterministic in (seed, round) -- re-runs each cell capped at
the reference's round count: that objective must equal the reference's bit
for bit (the B200 reaches the reference's 60-s solution after the same
rounds), and the 60-s GPU objective is the quality at equal wall time.
Writes profiles/r02_paper_scale.json.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "paper_scale_cpu.json")

mode = sys.argv[1]
n_inst = int(sys.argv[2]) if len(sys.argv) > 2 else 4
t_max = float(sys.argv[3]) if len(sys.argv) > 3 else 60.0
first = int(sys.argv[4]) if len(sys.argv) > 4 else 0   # cpu: append instances first..

if mode == "cpu":
    import remlot as pkg
    assert "/root/reference" in os.path.dirname(pkg.__file__), pkg.__file__
    from remlot import _kernels
    _kernels.warm_up()
else:
    sys.path.insert(0, ROOT)
    import paper_1704_05132_b200 as pkg

from dataclasses import replace  # noqa: E402

SCHEMES = pkg.SCHEMES


def cell(inst, scheme, **kw):
    cfg = pkg.SolverConfig(t_max=kw.pop("t_max", t_max), workers=2, seed=1, scheme=scheme,
                           **kw)
    t0 = time.monotonic()
    r = pkg.solve_scheme(inst, cfg)
    return dict(cost=int(r.cost), rounds=int(r.rounds), wall_s=round(time.monotonic() - t0, 3))


out = {"t_max": t_max, "instances": {}}
gold = None
if mode == "gpu":
    with open(GOLD) as f:
        gold = json.load(f)
    n_inst = min(n_inst, len(gold["instances"]))
elif first and os.path.exists(GOLD):
    with open(GOLD) as f:
        out = json.load(f)   # append to the earlier cells
for i in range(first, n_inst):
    name = f"gen{2000 + i}"
    inst = pkg.generate_instance(pkg.GeneratorConfig(products=300, periods=52, seed=2000 + i))
    row = {}
    for scheme in SCHEMES:
        if mode == "cpu":
            row[scheme] = cell(inst, scheme)
        else:
            pkg.solve_scheme(inst, pkg.SolverConfig(t_max=0.5, workers=2, seed=1, scheme=scheme,
                                                    max_rounds=2))   # module/graph warm-up
            g = gold["instances"][name][scheme]
            eq = cell(inst, scheme)
            capped = cell(inst, scheme, t_max=1e9, max_rounds=max(g["rounds"], 1)) \
                if scheme != "serial-vnd" else eq
            row[scheme] = dict(equal_time=eq, reference=g,
                               at_reference_rounds=capped,
                               bit_exact_at_reference_rounds=capped["cost"] == g["cost"],
                               rounds_ratio=eq["rounds"] / max(g["rounds"], 1))
        print(name, scheme, json.dumps(row[scheme]), flush=True)
    out["instances"][name] = row
if mode == "cpu":
    out["host"] = {"cores": len(os.sched_getaffinity(0)), "impl": "live reference (numba)"}
    with open(GOLD, "w") as f:
        json.dump(out, f, indent=1)
else:
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "r02_paper_scale.json"), "w") as f:
        json.dump(out, f, indent=1)
