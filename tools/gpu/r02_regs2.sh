L=gpurun_out/r02_regs2.log
for wl in c3 t63 c2; do for lib in cur m6 m8 r24 r8; do
  if [ $lib = cur ]; then unset REMLOT_B200_LIB; else export REMLOT_B200_LIB=paper_1704_05132_b200/_lib/libremlot_b200_$lib.so; fi
  timeout 120 python tools/ab_vnd.py $wl 0 | sed "s/^/$lib /" >> $L 2>&1
done; done
