L=gpurun_out/r02_tests2.log
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 >> $L
REMLOT_B200_LIB=$PWD/paper_1704_05132_b200/_lib/libremlot_b200_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_gvns.py -x -q 2>&1 | tail -3 >> $L
