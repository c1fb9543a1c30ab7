for i in 1 2; do for lib in "" m5 m6 m8; do for wl in c3 c2; do
  if [ -z "$lib" ]; then python tools/ab_vnd.py $wl 0 | sed "s/^/m7: /"; else REMLOT_B200_LIB=$PWD/paper_1704_05132_b200/_lib/libremlot_b200_$lib.so python tools/ab_vnd.py $wl 0 | sed "s/^/$lib: /"; fi
done; done; done >> gpurun_out/r02_regab.log 2>&1
