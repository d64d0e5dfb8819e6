#!/bin/bash
# Interleaved timing of several library builds: tools/ab_libs.sh "m n" reps lib1.so lib2.so ...
cd "$(dirname "$0")/.."
sz=$1; reps=$2; shift 2
for i in $(seq $reps); do
  for lib in "$@"; do
    printf "%-22s " "$(basename $lib)"
    SCQR3_LIB=$lib python tools/trsm_bench.py $sz --only trsm | tr '\n' ' '
    nvidia-smi --query-gpu=clocks.sm --format=csv,noheader | tr '\n' ' '
    echo
  done
done
