python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py -x -q 2>&1 | tail -3 > gpurun_out/r02_pf_tests.log
for i in 1 2; do for wl in c4; do
  python tools/ab_vnd.py $wl 0 2 | sed "s/^/new: /" >> gpurun_out/r02_pf_ab.log 2>&1
  REMLOT_B200_LIB=$PWD/paper_1704_05132_b200/_lib/libremlot_b200_ab.so python tools/ab_vnd.py $wl 0 2 | sed "s/^/old: /" >> gpurun_out/r02_pf_ab.log 2>&1
done; done
