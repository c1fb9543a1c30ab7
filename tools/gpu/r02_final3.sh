# final evidence after the e2e pipeline changes: bench line + launch list + GPU suite
python bench.py > gpurun_out/f3_bench.json 2> gpurun_out/f3_bench.err
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/f3_pytest_gpu.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/f3_launches_e2e_c3.csv python tools/profile_e2e.py > gpurun_out/f3_le.log 2>&1
