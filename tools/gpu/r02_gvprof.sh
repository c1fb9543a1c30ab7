ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_gvns_c2.csv python tools/profile_gvns.py 2 200 > gpurun_out/gv_l.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_shake|k_gvns_vnd' -s 10 -c 4 -o gpurun_out/r02_gvns python tools/profile_gvns.py 2 40 > gpurun_out/gv_f.log 2>&1
