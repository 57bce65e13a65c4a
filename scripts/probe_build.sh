#!/bin/bash
# Build a probe variant of one CUDA source into probe/probe_<name>.so (profiling only).
# usage: bash scripts/probe_build.sh <source.cu> "name:-DFLAG=1 ..." ...
set -e
SRC=$1; shift
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
mkdir -p build probe
base=$(basename $SRC)
OBJS=$(ls build/*.cu.o | grep -v "/$base.o")
for v in "$@"; do
  name=${v%%:*}; defs=${v#*:}
  nvcc $F $defs -c paper_2503_22879_b200/csrc/$SRC -o probe/probe_$name.o &
done
wait
for v in "$@"; do
  name=${v%%:*}
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o probe/probe_$name.so $OBJS probe/probe_$name.o
done
