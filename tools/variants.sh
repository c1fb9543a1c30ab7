#!/bin/bash
# Build k_vnd occupancy variants and time C3/C4 with each (dev experiment).
set -e
for minb in "$@"; do
  out=paper_1704_05132_b200/_lib/libremlot_b200_minb$minb.so
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
     -Xcompiler -fPIC -shared -DRL_VND_MINB=$minb -o $out paper_1704_05132_b200/csrc/remlot_b200.cu &
done
wait
for minb in "$@"; do
  echo "== minb $minb"
  REMLOT_B200_LIB=$PWD/paper_1704_05132_b200/_lib/libremlot_b200_minb$minb.so python tools/quick_time.py
done
