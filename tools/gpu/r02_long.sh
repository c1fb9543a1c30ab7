timeout 900 python -m pytest tests/test_gpu_pins.py -q -x -k long 2>&1 | tail -15 > gpurun_out/r02_long.log
