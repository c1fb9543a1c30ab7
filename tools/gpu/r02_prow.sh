L=gpurun_out/r02_prow.log
timeout 900 python -m pytest tests/test_gpu_gvns.py tests/test_gpu_pins.py -q -x -k "gvns or c5" 2>&1 | tail -2 >> $L
for i in 1 2; do for lib in base cur; do
  if [ $lib = cur ]; then unset REMLOT_B200_LIB; else export REMLOT_B200_LIB=paper_1704_05132_b200/_lib/libremlot_b200_$lib.so; fi
  for w in "2 400" "2 20000" "128 200" "1024 40"; do timeout 120 python tools/profile_gvns.py $w | sed "s/^/$lib /" >> $L 2>&1; done
done; done
