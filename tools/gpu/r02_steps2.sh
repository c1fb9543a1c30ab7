L=gpurun_out/r02_steps2.log
for wl in c3 c4 c2 t63; do for i in 1 2; do
  timeout 120 python tools/ab_vnd.py $wl 0 >> $L 2>&1
  REMLOT_B200_LIB=paper_1704_05132_b200/_lib/libremlot_b200_steps2.so timeout 120 python tools/ab_vnd.py $wl 0 | sed 's/^/steps2 /' >> $L 2>&1
done; done
