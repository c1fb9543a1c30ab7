"""Aggregate an ncu SASS source page by CUDA source line.

    ncu -i rep --page source --csv --print-source sass > sass.csv
    nvdisasm -g -c <cubin> > all.sass
    python tools/ncu_lines.py sass.csv all.sass <mangled kernel name> [top]
"""
import csv
import re
import sys
from collections import defaultdict

sass_csv, dis, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(dis).read().split("\n")
addr2src = {}
cur = None
inside = False
for l in lines:
    if l.startswith(".text.") and kname in l:
        inside = True
        continue
    if inside and l.startswith(".text.") and kname not in l:
        break
    if not inside:
        continue
    m = re.match(r'\s*//## File "(.*)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        addr2src[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
agg = defaultdict(lambda: [0, 0, 0, 0])
base = None
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        a = int(r[ix["Address"]], 16)
    except ValueError:
        continue
    if base is None:
        base = a
    a -= base
    src = addr2src.get(a, ("?", 0))
    g = agg[src]
    g[0] += int(r[ix["Instructions Executed"]] or 0)
    g[1] += int(r[ix["Thread Instructions Executed"]] or 0)
    g[2] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    g[3] += 1
tot = [sum(v[i] for v in agg.values()) for i in range(3)]
print(f"total warp inst {tot[0]:.3e} thread inst {tot[1]:.3e} samples {tot[2]}")
for src, v in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
    print(f"{src[0]:>16}:{src[1]:<5} inst {100*v[0]/tot[0]:5.1f}%  thr/inst {v[1]/max(v[0],1):5.1f}  "
          f"stall {100*v[2]/tot[2]:5.1f}%  sass {v[3]}")
