L=gpurun_out/r02_pvreg.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py tests/test_gpu_gvns.py tests/test_gpu_api.py -q -x 2>&1 | tail -2 >> $L
for i in 1 2; do for wl in c3 t63 c2; do for lib in base cur; do
  if [ $lib = cur ]; then unset REMLOT_B200_LIB; else export REMLOT_B200_LIB=paper_1704_05132_b200/_lib/libremlot_b200_$lib.so; fi
  timeout 120 python tools/ab_vnd.py $wl 0 | sed "s/^/$lib /" >> $L 2>&1
done; done; done
