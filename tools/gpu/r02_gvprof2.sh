ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_gvns_c2_v2.csv python tools/profile_gvns.py 2 200 > gpurun_out/r02_gvprof2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_gvns_c5_v2.csv python tools/profile_gvns.py 1024 10 >> gpurun_out/r02_gvprof2.log 2>&1
