L=gpurun_out/r02_setupfmt.log
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 >> $L
for wl in c3 c4 c2; do timeout 120 python tools/ab_vnd.py $wl 0 >> $L 2>&1; done
