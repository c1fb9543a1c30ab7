L=gpurun_out/r02_nw.log
for i in 1 2; do for nw in 4 3 2; do
  RL_NW_PER_CTA=$nw timeout 120 python tools/ab_vnd.py c4 0 | sed "s/^/nw$nw /" >> $L 2>&1
  RL_NW_PER_CTA=$nw timeout 120 python tools/ab_vnd.py c3 0 | sed "s/^/nw$nw /" >> $L 2>&1
done; done
