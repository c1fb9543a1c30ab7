# final evidence of HEAD (round 2)
python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/fin_pytest_gpu.log
bash tools/debug_checks.sh > gpurun_out/fin_debug_checks.log 2>&1; echo "rc=$?" >> gpurun_out/fin_debug_checks.log
python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
RL_BENCH_BACKEND=gloo python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fin_bench_n2.json 2> gpurun_out/fin_bench_n2.err
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'^void k_vnd<' -c 1 -o gpurun_out/fin_k_vnd_c3 python tools/profile_vnd.py c3 > gpurun_out/fin_ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'^void k_vnd<' -c 1 -o gpurun_out/fin_k_vnd_c4 python tools/profile_vnd.py c4 > gpurun_out/fin_ncu_c4.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/fin_ncu_bench.log 2>&1
