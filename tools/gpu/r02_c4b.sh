python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py -x -q 2>&1 | tail -5 > gpurun_out/r02_c4_tests.log
python tools/ab_vnd.py c4 0 128 2 > gpurun_out/r02_c4_ab.log 2>&1
