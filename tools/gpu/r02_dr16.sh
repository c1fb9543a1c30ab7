L=gpurun_out/r02_dr16.log
REMLOT_B200_LIB=paper_1704_05132_b200/_lib/libremlot_b200_dr16.so timeout 900 python -m pytest tests/test_gpu_pins.py -q -x -k "c4 or long" 2>&1 | tail -1 >> $L
for i in 1 2; do for wl in c4 t200; do for lib in cur dr16; do
  if [ $lib = cur ]; then unset REMLOT_B200_LIB; else export REMLOT_B200_LIB=paper_1704_05132_b200/_lib/libremlot_b200_$lib.so; fi
  timeout 120 python tools/ab_vnd.py $wl 0 | sed "s/^/$lib /" >> $L 2>&1
done; done; done
