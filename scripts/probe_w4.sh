#!/bin/bash
# Build timing-probe variants of the W4A8 GEMM into probe/probe_<name>.so (profiling only).
# usage: bash scripts/probe_w4.sh "name:-DFLAG=1 ..." ...   (then python scripts/probe_w4.py name ...)
set -e
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
mkdir -p build probe
OBJS=$(ls build/*.cu.o | grep -v gemm_w4a8)
for v in "$@"; do
  name=${v%%:*}; defs=${v#*:}
  nvcc $F $defs -c paper_2503_22879_b200/csrc/gemm_w4a8.cu -o probe/probe_$name.o &
done
wait
for v in "$@"; do
  name=${v%%:*}
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o probe/probe_$name.so $OBJS probe/probe_$name.o
done
