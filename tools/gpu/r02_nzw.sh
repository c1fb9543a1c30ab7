L=gpurun_out/r02_nzw.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py -q -x -k "fuzz or long_horizon or t520 or c4 or wide or t130" 2>&1 | tail -2 >> $L
for i in 1 2; do for wl in c4 t200; do for lib in base nzw; do
  REMLOT_B200_LIB=paper_1704_05132_b200/_lib/libremlot_b200_$lib.so timeout 120 python tools/ab_vnd.py $wl 0 | sed "s/^/$lib /" >> $L 2>&1
done; done; done
