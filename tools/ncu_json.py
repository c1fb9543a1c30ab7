"""Write the bench-facing summaries of an ncu --set full capture of k_vnd:

    python tools/ncu_json.py gpurun_out/c3_full.ncu-rep c3 r01

-> profiles/k_vnd_<wl>_traffic.json (dram bytes per launch, bench roofline
   'traffic') and profiles/k_vnd_<wl>_ncu.json (issue-slot, pipe and SIMT
   utilisation: bench roofline 'ncu').
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, wl, rnd = sys.argv[1:4]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
kcol = hdr.index("Kernel Name")
# the VND kernel's row (a capture may hold other launches too)
vals = next((r for r in rows[2:] if r[kcol].startswith("void k_vnd<")), rows[2])
get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(name, scale=1.0):
    v, u = get[name]
    x = float(v.replace(",", ""))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3,
            "ms": 1.0, "s": 1e3}.get(u, 1.0)
    return x * mult * scale


kname = get["Kernel Name"][0] if "Kernel Name" in get else ""
rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
src = f"profiles/{rnd}_k_vnd_{wl}_ncu.txt (ncu --set full --clock-control none)"
traffic = {"bytes_per_launch": int(rd + wr), "dram_read_MB": round(rd / 1e6, 2),
           "dram_write_MB": round(wr / 1e6, 2), "source": src, "kernel": kname}
summary = {
    "source": src, "kernel": kname,
    "duration_ms": round(num("gpu__time_duration.sum"), 3),
    "issue_active_pct": round(num("smsp__issue_active.avg.pct_of_peak_sustained_active"), 1),
    "alu_pipe_pct": round(num("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"), 1),
    "fma_pipe_pct": round(num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"), 1),
    "threads_per_inst": round(num("smsp__thread_inst_executed_per_inst_executed.ratio"), 2),
    "threads_pred_on_per_inst": round(
        num("smsp__thread_inst_executed_pred_on_per_inst_executed.ratio"), 2),
    "sm_clock_mhz": round(float(get["sm__cycles_elapsed.avg.per_second"][0].replace(",", "")) * {
        "Ghz": 1e3, "GHz": 1e3, "Mhz": 1.0, "MHz": 1.0, "hz": 1e-6, "Hz": 1e-6}.get(
        get["sm__cycles_elapsed.avg.per_second"][1], 1.0), 1),
    "warps_active_pct": round(num("sm__warps_active.avg.pct_of_peak_sustained_active"), 1),
    "warp_inst": int(num("smsp__inst_executed.sum")),
    "registers": int(num("launch__registers_per_thread")),
    "smem_wavefronts": int(num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")),
    "smem_pipe_pct": round(
        num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"), 1),
    "dram_gbs": round((rd + wr) / (num("gpu__time_duration.sum") * 1e-3) / 1e9, 2),
}
for name, obj in (("traffic", traffic), ("ncu", summary)):
    path = os.path.join(ROOT, "profiles", f"k_vnd_{wl}_{name}.json")
    with open(path, "w") as f:
        json.dump(obj, f, indent=1)
    print(path, json.dumps(obj))
