#!/bin/bash
# interleaved TRSM timings of variant libraries: tools/_ab_diag.sh "m n" reps diag lib...
cd "$(dirname "$0")/.."
sz=$1; reps=$2; diag=$3; shift 3
for i in $(seq $reps); do
  for lib in "$@"; do
    printf "%-12s " "$(basename $lib)"
    SCQR3_LIB=$lib python tools/trsm_bench.py $sz --only trsm --diag $diag | tr '\n' ' '
    echo
  done
done
