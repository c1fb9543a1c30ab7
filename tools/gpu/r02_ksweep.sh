for wl in c2 k12k k25k k50k c3 k200k; do python tools/ab_vnd.py $wl 0 >> gpurun_out/r02_ksweep.log 2>&1; done
