L=gpurun_out/r02_chunks.log
for lib in cur ch3 ch6 ch8; do
  if [ $lib = cur ]; then unset REMLOT_B200_LIB; else export REMLOT_B200_LIB=paper_1704_05132_b200/_lib/libremlot_b200_$lib.so; fi
  timeout 300 python tools/e2e_compare.py 100000 52 10 | sed "s/^/$lib /" >> $L 2>&1
done
