"""Summarise ncu outputs (launch list CSV, --set full report) into profiles/ (tracked).

  python tools/summarize_ncu.py --launches gpurun_out/launches_r01.csv \
      --full gpurun_out/prof_bench_r01.ncu-rep --round r01 --config C3
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    # a list captured with `--kernel-name-base demangled -k regex:scqr3` holds only the library's
    # kernels, printed without the namespace
    filtered = not any("scqr3::" in r[ki] for r in rows[h + 1:] if len(r) > ki)
    for r in rows[h + 1:]:
        if len(r) <= ki or (not filtered and "scqr3::" not in r[ki]):
            continue  # input generation (torch / cuSOLVER) is not part of the step
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0].replace("scqr3::", "")
        tot[name] += float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1e-6)
        cnt[name] += 1
    T = sum(tot.values())
    return {k: {"launches": cnt[k], "total_ms": tot[k], "avg_ms": tot[k] / cnt[k], "share": tot[k] / T}
            for k in sorted(tot, key=lambda k: -tot[k])}


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    res = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("scqr3::", "")
        d = {}
        for w in want:
            if w in hdr:
                i = hdr.index(w)
                d[w] = {"value": r[i], "unit": units[i]}
        res.setdefault(name, d)
    return res


def gbytes(v):
    x = float(v["value"].replace(",", ""))
    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(v["unit"], 1.0)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--round", default="r01")
    ap.add_argument("--config", default="C3")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    out_path = os.path.join(PROF, f"ncu_{a.round}_{a.config}.json")
    summary = json.load(open(out_path)) if os.path.exists(out_path) else {}  # keep the other part
    summary.update({"config": a.config, "round": a.round})
    if a.launches:
        summary["launch_list"] = launches(a.launches)
        summary["launch_list_note"] = ("ncu --metrics gpu__time_duration.sum --clock-control none: per-launch "
                                       "device times, cold-cache and serialised; compare SHARES with bench.py")
    if a.full:
        f = full(a.full)
        summary["full"] = f
        traffic_path = os.path.join(PROF, "ncu_traffic.json")
        traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
        seen = {}
        for name, d in f.items():
            key = "gram" if name.startswith("gram") else "trsm" if name.startswith("trsm") else name
            by = gbytes(d["dram__bytes_read.sum"]) + gbytes(d["dram__bytes_write.sum"])
            if by < seen.get(key, 0.0):
                continue  # (the TRSM's twin instance that reads the guard flag and exits at once)
            seen[key] = by
            traffic[f"{a.config}:{key}"] = {
                "bytes_per_launch": by,
                "source": f"profiles/ncu_{a.round}_{a.config}.json (ncu --set full, one launch)"}
        json.dump(traffic, open(traffic_path, "w"), indent=1)
    json.dump(summary, open(out_path, "w"), indent=1)
    print(json.dumps(summary, indent=1)[:3000])
