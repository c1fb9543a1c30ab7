#!/bin/bash
# Build the library with device bounds asserts (-DRL_DEBUG_CHECKS) and run the
# sanitizer workload and the GPU tests against it (compute-sanitizer is not
# available on this pool).
set -e
out=paper_1704_05132_b200/_lib/libremlot_b200_debug.so
# built here when missing or older than the sources (prebuild it in the build
# container: nvcc needs no GPU)
if [ ! -f $out ] || [ -n "$(find paper_1704_05132_b200/csrc include -newer $out -type f)" ]; then
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
     -Xcompiler -fPIC -shared -DRL_DEBUG_CHECKS -o $out paper_1704_05132_b200/csrc/remlot_b200.cu
fi
export REMLOT_B200_LIB=$PWD/$out
python tools/sanitize_run.py
python -m pytest tests -m gpu -q -x
