#!/bin/bash
# A/B of the CSR Y = BQ kernels (SCQR3_CSR_Y=0: thread per (row, 16-column chunk); 1..6: 256-row
# tile kernel instances) on C5L: parity tests of every variant, then the bench line of each.
out=${1:-gpurun_out/csry}
mkdir -p $out
for v in ${VARIANTS:-0 1 2 3 4 5 6}; do
  SCQR3_CSR_Y=$v timeout 600 python -m pytest ${TESTS:-tests} -m gpu -q -x -k "csr or ghost or laplacian" > $out/test_v$v.log 2>&1
  echo "variant $v tests: $(tail -1 $out/test_v$v.log)"
  SCQR3_CSR_Y=$v timeout 600 python bench.py --config C5L --steps 5 --warmup 3 --no-cpu --no-e2e > $out/bench_v$v.json 2> $out/bench_v$v.err
  python - $out/bench_v$v.json $v <<'P'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k = d["kernels"]
print("variant", sys.argv[2], "ms_per_step", round(d["ms_per_step"], 3), "passes", d.get("passes"),
      "y+reduce avg ms", round(k["reduce"]["avg_ms"] * 2, 4), "gram", round(k["gram"]["avg_ms"], 4),
      "trsm", round(k["trsm"]["avg_ms"], 4))
P
done
