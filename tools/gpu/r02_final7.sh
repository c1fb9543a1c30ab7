# final evidence at HEAD (dense-pass previous-setup table): ncu C3 + C4, bench line, launch list
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'^void k_vnd<' -c 1 -o gpurun_out/f7_k_vnd_c3 python tools/profile_vnd.py c3 > gpurun_out/f7_ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'^void k_vnd<' -c 1 -o gpurun_out/f7_k_vnd_c4 python tools/profile_vnd.py c4 > gpurun_out/f7_ncu_c4.log 2>&1
python tools/ncu_json.py gpurun_out/f7_k_vnd_c3.ncu-rep c3 r02 > gpurun_out/f7_ncu_json.log 2>&1
python tools/ncu_json.py gpurun_out/f7_k_vnd_c4.ncu-rep c4 r02 >> gpurun_out/f7_ncu_json.log 2>&1
cp profiles/k_vnd_c3_ncu.json profiles/k_vnd_c3_traffic.json profiles/k_vnd_c4_ncu.json profiles/k_vnd_c4_traffic.json gpurun_out/
python bench.py > gpurun_out/f7_bench.json 2> gpurun_out/f7_bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/f7_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/f7_ncu_bench.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/f7_pytest_gpu.log
