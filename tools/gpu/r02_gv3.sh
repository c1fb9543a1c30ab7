python -m pytest tests/test_gpu_gvns.py tests/test_gpu_concurrency.py tests/test_gpu_pins.py tests/test_gpu_api.py -q -x 2>&1 | tail -6 > gpurun_out/r02_gv_tests.log
for w in "2 400" "2 20000" "16 2000" "128 200" "1024 40"; do python tools/profile_gvns.py $w >> gpurun_out/r02_gv_rate.log 2>&1; done
