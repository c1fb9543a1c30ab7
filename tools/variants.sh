#!/bin/bash
# Build compile-time variants of the library and time them (dev experiment).
#   AB_CONFIGS=c3,c4 tools/variants.sh "-DRL_REFILL_MIN=8" "-DRL_VND_MINB=5" ...
set -e
i=0
for flags in "$@"; do
  out=paper_1704_05132_b200/_lib/libremlot_b200_v$i.so
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
     -Xcompiler -fPIC -shared $flags -o $out paper_1704_05132_b200/csrc/remlot_b200.cu &
  i=$((i+1))
done
wait
i=0
for flags in "$@"; do
  echo "== variant $i: $flags"
  REMLOT_B200_LIB=$PWD/paper_1704_05132_b200/_lib/libremlot_b200_v$i.so python tools/ab.py ${AB_CONFIGS:-c2,c3,c4} 0 3
  i=$((i+1))
done
