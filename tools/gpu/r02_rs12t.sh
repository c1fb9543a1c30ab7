L=gpurun_out/r02_rs12t.log
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 >> $L
for i in 1 2; do timeout 120 python tools/ab_vnd.py c4 0 >> $L 2>&1; done
