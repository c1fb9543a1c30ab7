python -m pytest tests/test_gpu_gvns.py tests/test_gpu_concurrency.py tests/test_native_lib.py -q -x 2>&1 | tail -8 > gpurun_out/r02_gv_tests.log
