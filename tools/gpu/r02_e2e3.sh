L=gpurun_out/r02_e2e3.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_concurrency.py -q -x 2>&1 | tail -2 >> $L
timeout 300 python tools/e2e_compare.py 100000 52 10 >> $L 2>&1
