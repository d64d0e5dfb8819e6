#!/bin/bash
# End-of-session evidence run: full GPU suite, smoke, every config's bench line, the reference arm,
# ncu launch lists (C3, C5L) of the same bench command.  Output under $1 (default gpurun_out/final).
out=${1:-gpurun_out/final}
mkdir -p $out
python -m pytest tests -m gpu -x -q > $out/gputest.log 2>&1; echo "pytest rc=$?" >> $out/gputest.log
python __graft_entry__.py smoke > $out/smoke.log 2>&1
python bench.py > $out/bench_C3.json 2> $out/bench_C3.err
for c in C2 C5 C5L PR1; do python bench.py --config $c > $out/bench_$c.json 2> $out/bench_$c.err; done
python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_reference_arm.json 2> $out/bench_reference_arm.err
for c in C3 C5L; do
  ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:scqr3 --csv --log-file $out/ncu_launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 1 --no-cpu --no-e2e > $out/ncu_$c.log 2>&1
done
tail -2 $out/gputest.log; tail -1 $out/smoke.log
for c in C3 C2 C5 C5L PR1; do python - $out/bench_$c.json $c <<'P'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], "ms", round(d["ms_per_step"], 4), "TF/s", round(d["value"], 2), "roofline", round(d["roofline"]["frac"], 3),
      "step", round(d["roofline_step"]["frac"], 3) if d.get("roofline_step") else None, "e2e", d.get("e2e", {}).get("value"))
P
done
