#!/bin/bash
# Build the walk-statistics variant and print the delta-walk statistics.
set -e
out=paper_1704_05132_b200/_lib/libremlot_b200_walkstats.so
if [ ! -f $out ] || [ paper_1704_05132_b200/csrc/vnd_device.cuh -nt $out ]; then
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
     -Xcompiler -fPIC -shared -DRL_WALK_STATS -o $out paper_1704_05132_b200/csrc/remlot_b200.cu
fi
REMLOT_B200_LIB=$PWD/$out python tools/walk_stats.py "$@"  # RL_VARIANTS=0,4,8 to compare
