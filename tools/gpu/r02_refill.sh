for r in 8 12 24; do for wl in c3 c4; do REMLOT_B200_LIB=$PWD/paper_1704_05132_b200/_lib/libremlot_b200_r$r.so python tools/ab_vnd.py $wl 0 | sed "s/^/refill $r: /" >> gpurun_out/r02_refill.log 2>&1; done; done
for wl in c3 c4; do python tools/ab_vnd.py $wl 0 | sed "s/^/refill 16: /" >> gpurun_out/r02_refill.log 2>&1; done
