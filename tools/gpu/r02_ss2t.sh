L=gpurun_out/r02_ss2t.log
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 >> $L
