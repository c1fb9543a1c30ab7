L=gpurun_out/r02_steps.log
for wl in c3 t63 c4 c2; do for lib in s2 s3 s4 s2r12 s2r20; do
  REMLOT_B200_LIB=paper_1704_05132_b200/_lib/libremlot_b200_$lib.so timeout 120 python tools/ab_vnd.py $wl 0 | sed "s/^/$lib /" >> $L 2>&1
done; done
for lib in base s2 s3; do
  for w in "2 20000" "128 200" "1024 40"; do
  REMLOT_B200_LIB=paper_1704_05132_b200/_lib/libremlot_b200_$lib.so timeout 120 python tools/profile_gvns.py $w | sed "s/^/$lib /" >> $L 2>&1
  done
done
