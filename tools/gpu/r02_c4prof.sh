python -m pytest tests/test_gpu_reference_suite.py tests/test_gpu_pins.py -m gpu -q -rs 2>&1 | tail -8 > gpurun_out/r02_skips.log
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'^void k_vnd<' -c 1 -o gpurun_out/r02_k_vnd_c4p16 python tools/profile_vnd.py c4 > gpurun_out/ncu_c4.log 2>&1
