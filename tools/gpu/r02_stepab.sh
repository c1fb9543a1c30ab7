python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/r02_step_tests.log
for wl in c3 c4 c2; do
  python tools/ab_vnd.py $wl 0 0 >> gpurun_out/r02_step_ab.log 2>&1
  REMLOT_B200_LIB=$PWD/paper_1704_05132_b200/_lib/libremlot_b200_ab.so python tools/ab_vnd.py $wl 0 0 | sed 's/^/branch: /' >> gpurun_out/r02_step_ab.log 2>&1
done
