set -x
nvidia-smi -L
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r02_pytest_gpu.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench0.json 2> gpurun_out/r02_bench0.err
ncu --set full --clock-control none --import-source on -k regex:k_vnd -s 1 -c 1 -o gpurun_out/r02_c3_head python tools/profile_vnd.py c3 > gpurun_out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_vnd -s 1 -c 1 -o gpurun_out/r02_c4_head python tools/profile_vnd.py c4 > gpurun_out/ncu_c4.log 2>&1
ls -la gpurun_out
