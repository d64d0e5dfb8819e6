"""Aggregate an ncu report's per-instruction warp-stall samples by CUDA source line:
python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = None
cur = None
agg = defaultdict(float)
reasons = defaultdict(lambda: defaultdict(float))
src = {}
for r in rows:
    if r and r[0] == "Line No":
        h = r
        ix = {}
        for i, k in enumerate(h):
            ix.setdefault(k, i)
        samp = ix["Warp Stall Sampling (All Samples)"]
        stalls = [k for k in h if k.startswith("stall_") and "Not" not in k]
        continue
    if h is None or len(r) < 4 or r[0] in ("File Path", "Function Name"):
        continue
    if r[0]:
        try:
            cur = int(r[0])
        except ValueError:
            continue
        src[cur] = r[1]
        continue
    if len(r) > samp and r[samp] not in ("", "-"):
        try:
            v = float(r[samp])
        except ValueError:
            continue
        agg[cur] += v
        for k in stalls:
            try:
                reasons[cur][k] += float(r[ix[k]] or 0)
            except (ValueError, IndexError):
                pass
tot = sum(agg.values())
tr = defaultdict(float)
for line in reasons:
    for k, v in reasons[line].items():
        tr[k] += v
print(f"total samples {tot:.0f}; by reason:",
      ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(tr.items(), key=lambda x: -x[1])[:8]))
for line, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    t3 = sorted(reasons[line].items(), key=lambda x: -x[1])[:3]
    print(f"{v:6.0f} {100 * v / tot:5.1f}% L{line:4d} {src.get(line, '?').strip()[:64]:64s} "
          f"{[(k[6:], int(x)) for k, x in t3]}")
