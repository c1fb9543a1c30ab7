#!/bin/bash
# Summarise an ncu report of k_vnd: headline metrics + hottest source lines.
#   tools/ncu_report.sh gpurun_out/prof.ncu-rep [mangled-kernel-prefix]
rep=$1; kern=${2:-_Z5k_vndIiiN2rl7MaskRegEEv}
ncu -i "$rep" --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]; v=rows[2]
for w in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','smsp__thread_inst_executed_per_inst_executed.ratio','sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']:
    for i,x in enumerate(h):
        if x==w: print(f'{w:60s} {rows[1][i]:>8s} {v[i]}')
"
tmp=$(mktemp -d)
lib=$(realpath $(dirname $0)/../paper_1704_05132_b200/_lib/libremlot_b200.so); (cd $tmp && cuobjdump -xelf all $lib >/dev/null 2>&1 && nvdisasm -g -c *.cubin > all.sass 2>/dev/null)
ncu -i "$rep" --page source --csv --print-source sass 2>/dev/null > $tmp/sass.csv
python3 $(dirname $0)/ncu_lines.py $tmp/sass.csv $tmp/all.sass $kern ${3:-30} | python3 -c "
import re,sys,os
root=os.path.join('$(dirname $0)','..','paper_1704_05132_b200','csrc')
cache={}
for l in sys.stdin:
    m=re.match(r'\s*(\S+):(\d+)\s',l)
    if m and os.path.exists(os.path.join(root,m.group(1))):
        f=m.group(1)
        cache.setdefault(f, open(os.path.join(root,f)).read().split('\n'))
        print(l.rstrip()[:96], '|', cache[f][int(m.group(2))-1].strip()[:56])
    else: print(l.rstrip())
"
rm -rf $tmp
