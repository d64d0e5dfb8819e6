#!/bin/bash
# A/B of tridiagonal Y = BQ kernel builds on C5 (tools/build_variant.sh NAME gram.cu -D...):
# oblique parity tests, then the C5 bench line of each library.
out=${1:-gpurun_out/yab}
mkdir -p $out
for v in base ${VARIANTS:-yfast4 yfast8 yfast2}; do
  lib=""; [ $v != base ] && lib=$PWD/_variants/$v.so
  SCQR3_LIB=$lib timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "oblique" > $out/test_$v.log 2>&1
  echo "$v tests: $(tail -1 $out/test_$v.log)"
  SCQR3_LIB=$lib timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > $out/bench_$v.json 2> $out/bench_$v.err
  python - $out/bench_$v.json $v <<'P'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k = d["kernels"]
print(sys.argv[2], "ms_per_step", round(d["ms_per_step"], 3), "y+reduce avg ms", round(k["reduce"]["avg_ms"] * 2, 4),
      "gram", round(k["gram"]["avg_ms"], 4), "trsm", round(k["trsm"]["avg_ms"], 4))
P
done
