#!/bin/bash
# Interleaved A/B timing of the C3 TRSM/Gram kernels: tools/ab_trsm.sh libA.so libB.so [reps]
cd "$(dirname "$0")/.."
reps=${3:-3}
for i in $(seq $reps); do
  for lib in "$1" "$2"; do
    printf "%-28s " "$(basename $lib)"
    SCQR3_LIB=$lib python tools/trsm_bench.py 10000000 128 | tr '\n' ' '
    nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu --format=csv,noheader | tr '\n' ' '
    echo
  done
done
