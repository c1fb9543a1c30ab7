python -m pytest tests/test_gpu_gvns.py tests/test_gpu_pins.py -q -x -k "gvns or c5 or shake or worker" 2>&1 | tail -2 > gpurun_out/r02_gminb_tests.log
for lib in "" g6 g4; do for w in "2 400" "2 20000" "128 200" "1024 40"; do
  if [ -z "$lib" ]; then python tools/profile_gvns.py $w | sed "s/^/minb7: /"; else REMLOT_B200_LIB=$PWD/paper_1704_05132_b200/_lib/libremlot_b200_$lib.so python tools/profile_gvns.py $w | sed "s/^/$lib: /"; fi
done; done >> gpurun_out/r02_gminb.log 2>&1
