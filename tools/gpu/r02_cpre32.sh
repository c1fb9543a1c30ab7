L=gpurun_out/r02_cpre32b.log
for kt in "64 520 2" "1000 520 0" "3000 200 0"; do
  timeout 60 python tools/hang_probe.py $kt >> $L 2>&1 || { echo "rc=$? $kt" >> $L; exit 1; }
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cpre32 or int32_coefficient or t520 or long_horizon or fuzz" 2>&1 | tail -3 >> $L
timeout 600 python -m pytest tests/test_gpu_pins.py -q -x -k "c4" 2>&1 | tail -3 >> $L
for i in 1 2; do
REMLOT_B200_LIB=paper_1704_05132_b200/_lib/libremlot_b200_base.so timeout 120 python tools/ab_vnd.py c4 0 >> $L 2>&1
timeout 120 python tools/ab_vnd.py c4 0 128 >> $L 2>&1
done
