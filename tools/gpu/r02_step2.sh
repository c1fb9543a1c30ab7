python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r02_step_tests.log
REMLOT_B200_LIB=$PWD/paper_1704_05132_b200/_lib/libremlot_b200_debug.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q 2>&1 | tail -3 >> gpurun_out/r02_step_tests.log
for wl in c3 c4; do python tools/ab_vnd.py $wl 0 >> gpurun_out/r02_step_ab2.log 2>&1; done
