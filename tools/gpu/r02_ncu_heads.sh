ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'^void k_vnd<' -c 1 -o gpurun_out/r02_k_vnd_c3 python tools/profile_vnd.py c3 > gpurun_out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'^void k_vnd<' -c 1 -o gpurun_out/r02_k_vnd_c4 python tools/profile_vnd.py c4 > gpurun_out/ncu_c4.log 2>&1
