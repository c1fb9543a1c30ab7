python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2 > gpurun_out/r02_regab2_tests.log
for i in 1 2; do
  python tools/ab_vnd.py c2 0 | sed "s/^/new: /"
  python tools/ab_vnd.py c4 0 | sed "s/^/s5: /"
  REMLOT_B200_LIB=$PWD/paper_1704_05132_b200/_lib/libremlot_b200_s4.so python tools/ab_vnd.py c4 0 | sed "s/^/s4: /"
done >> gpurun_out/r02_regab2.log 2>&1
