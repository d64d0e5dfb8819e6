#!/bin/bash
# Build an experiment variant of libscqr3.so: tools/build_variant.sh NAME FILE.cu -DFLAG...
# (the other objects come from the in-tree build; select it with SCQR3_LIB=_variants/NAME.so)
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
B=paper_1809_11085_b200/_build
mkdir -p _variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Iinclude -Ipaper_1809_11085_b200/csrc "$@" -c paper_1809_11085_b200/csrc/$src -o _variants/$name.o
objs=""
for f in gram chol zchol zwide trsm comm scqr3_host; do
  if [ "$f.cu" = "$src" ]; then objs="$objs _variants/$name.o"; else objs="$objs $B/$f.o"; fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _variants/$name.so $objs -lnccl
echo _variants/$name.so
