# evidence of HEAD: ncu full captures (C3, C4), C3 launch list, default bench line
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'^void k_vnd<' -c 1 -o gpurun_out/ev_k_vnd_c3 python tools/profile_vnd.py c3 > gpurun_out/ev_ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'^void k_vnd<' -c 1 -o gpurun_out/ev_k_vnd_c4 python tools/profile_vnd.py c4 > gpurun_out/ev_ncu_c4.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev_launches_c3.csv python tools/profile_vnd.py c3 > gpurun_out/ev_l.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev_launches_e2e.csv python tools/profile_e2e.py > gpurun_out/ev_le.log 2>&1
