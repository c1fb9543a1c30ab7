L=gpurun_out/r02_chunks3.log
for i in 1 2; do for lib in cur c3r3 c3r4 c4r2 c2r2; do
  if [ $lib = cur ]; then unset REMLOT_B200_LIB; else export REMLOT_B200_LIB=paper_1704_05132_b200/_lib/libremlot_b200_$lib.so; fi
  timeout 300 python tools/e2e_compare.py 100000 52 10 2>&1 | grep "pipelined=True" | tail -1 | sed "s/^/$lib /" >> $L
done; done
