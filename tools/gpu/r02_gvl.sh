ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_gvns_c2.csv python tools/profile_gvns_batches.py 2 200 > gpurun_out/gv_l.log 2>&1
