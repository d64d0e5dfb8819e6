#!/usr/bin/env python
"""bench.py -- shifted CholeskyQR3 fp64 TFLOP/s and % of roofline (BASELINE.json metric).

Workload (BASELINE.json configs[2], the headline): X fp64 m = 10,000,000 x n = 128, kappa_2 = 1e10,
X = U diag(sigma) V^T with geometric sigma, seed 0, generated on the device.
One "step" = one full scqr3_factor call (every pass of Gram -> shifted Cholesky -> TRSM -> R
accumulation until the stop rule fires; 3 passes on this workload) through the C ABI.
value = 6 m n^2 / t (the north star's 3-pass flop count, whole job over all ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N    (one rank per GPU)

Rows are block-partitioned across ranks; each pass does one NCCL allreduce of the packed n x n
Gram (the method's one exchange): total work is fixed as N grows -> "strong" scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAKS = os.path.join(ROOT, "profiles", "fp64_peaks.json")
NCU_TRAFFIC = os.path.join(ROOT, "profiles", "ncu_traffic.json")
METRIC = "shifted CholeskyQR3 fp64 TFLOP/s & % roofline, m=1e7 n=128, 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C3")
    ap.add_argument("--m", type=int, default=0, help="override the config's m (exploration only)")
    ap.add_argument("--cpu-rows", type=int, default=0, help="rows of the oracle's bounded sample")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--force-comm", action="store_true",
                    help="use the NCCL communicator path even at one rank (exercises the multi-GPU code)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def flops_3pass(m, n):
    return 6.0 * m * n * n


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def executed_roofline_ms(cfg, m, n, passes, peak_tflops, fused, nnz=0, hbm_gbs=6536.7):
    """Roofline time of the work a factorisation executed on this rank: the sum over its kernels
    (which run one after another) of max(algorithmic flops / FP64 peak, algorithmic bytes / HBM
    bandwidth), for the executed pass count.  Per pass: Gram m n(n+1) flop, 8mn B (oblique: the
    dual B-Gram + plain Gram, 2 m n(n+1) flop, 16mn B, after Y = BQ: tridiagonal 5mn flop,
    16mn + 16m B; CSR 2 nnz n flop, 16mn + 12 nnz + 8m B: the CSR arrays once); TRSM m n^2 flop, 16mn B; the
    fused n <= 64 TRSM also carries the next pass's Gram (no 8mn re-read).  The n x n steps
    (reduce, Cholesky) are latency and not in the model."""
    P, BW = peak_tflops * 1e12, hbm_gbs * 1e9
    t = lambda fl, by: max(fl / P, by / BW)  # noqa: E731
    tot = 0.0
    for k in range(1, passes + 1):
        if cfg.oblique:
            if cfg.metric == "laplacian":
                tot += t(2.0 * nnz * n, 16.0 * m * n + 12.0 * nnz + 8.0 * m)
            else:
                tot += t(5.0 * m * n, 16.0 * m * n + 16.0 * m)
            tot += t(2.0 * m * n * (n + 1), 16.0 * m * n)
            tot += t(1.0 * m * n * n, 16.0 * m * n)
        elif fused:
            if k == 1:
                tot += t(1.0 * m * n * (n + 1), 8.0 * m * n)
            fl = m * n * n + (m * n * (n + 1) if k < passes else 0)
            tot += t(fl, 16.0 * m * n)
        else:
            tot += t(1.0 * m * n * (n + 1), 8.0 * m * n) + t(1.0 * m * n * n, 16.0 * m * n)
    model = ("sum over the executed kernels of max(flops / fp64 peak, bytes / 6536.7 GB/s), "
             f"{passes} passes, per GPU")
    return tot * 1e3, model


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
                power.append(float(p[3]))
            except ValueError:
                continue
            for name, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    import synth

    cfg = synth.CONFIGS[args.config]
    n = cfg.n
    rows = args.cpu_rows or max(n, int(2e6 * (128 / n) ** 2))  # ~4 s of oracle work per step (16 cores)
    rows = min(rows, cfg.m)
    kw = {}
    if cfg.oblique:
        kind, B, rows = synth.config_metric(cfg, rows)
        kw = dict(csr=B) if kind == "csr" else dict(d=B[0], e=B[1])
    X = synth.randsvd(rows, n, cfg.kappa, seed=0, spectrum=cfg.spectrum)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = oracle.scqr3(X, **kw)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t = statistics.mean(times)
    val = flops_3pass(rows, n) / t / 1e12
    cores = oracle.num_threads()
    sample = f"oracle.scqr3 on the first {rows} of {cfg.m} rows ({args.config} recipe, host numpy stream), per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} bounded sample: m={rows} n={n} kappa={cfg.kappa:g}",
                   "m": rows, "n": n, "passes": r.passes, "status": r.status},
        "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def host_mem_available():
    """MemAvailable of /proc/meminfo in bytes (0 if unreadable)."""
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return 1024.0 * float(line.split()[1])
    except OSError:
        pass
    return 0.0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1809_11085_b200 as sq
    from paper_1809_11085_b200 import _abi
    import synth

    rank, world, local = dist_env()
    multi = world > 1 or args.force_comm
    if multi and "RANK" not in os.environ:  # --force-comm without a launcher: a one-rank group
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=os.environ.get("MASTER_PORT", "29541"))
    if multi:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    cfg = synth.CONFIGS[args.config]
    m, n = (args.m or cfg.m), cfg.n
    if cfg.oblique and cfg.metric == "laplacian":
        m = max(cfg.grid_nx, (m // cfg.grid_nx) * cfg.grid_nx)   # whole grid lines
    from paper_1809_11085_b200.dist import row_block

    r0, r1 = row_block(m, rank, world)
    mloc = r1 - r0

    # ---- input: each rank generates only its own rows of the global X (per-chunk seeded TSQR
    # generator: the stitched X is the same for every rank count; synth.randsvd_torch_rows)
    X = synth.randsvd_torch_rows(m, n, cfg.kappa, r0, r1, seed=0, spectrum=cfg.spectrum, device=dev,
                                 allreduce=(dist.all_reduce if world > 1 else None))
    d = e = csr = None
    if cfg.oblique and cfg.metric == "laplacian":
        Bg = synth.laplacian2d(cfg.grid_nx, m // cfg.grid_nx, seed=0, wmax=1e4)
        csr = sq.CsrMetric(*synth.csr_rows(Bg, r0, r1), halo=cfg.grid_nx if world > 1 else 0, device=dev)
        del Bg
    elif cfg.oblique:
        dg, eg = synth.tridiag_b_torch(m, seed=0, device=dev)
        d, e = dg[r0:r1].contiguous(), eg[r0:r1].contiguous()
        del dg, eg
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    comm = sq.Comm.create() if multi else None
    stream = torch.cuda.Stream(device=dev)
    ws = (sq.workspace(mloc, n, device=dev, csr_halo=csr.halo) if csr is not None
          else sq.workspace(mloc, n, oblique=cfg.oblique, device=dev))
    Q = sq.colmajor_empty(mloc, n, device=dev)
    R = torch.empty((n, n), dtype=torch.float64, device=dev).t()
    prof = _abi.Prof()

    def step(with_prof=False):
        kw = dict(Q=Q, R=R, ws=ws, comm=comm, m_global=m, stream=stream)
        if with_prof:
            kw["prof"] = prof
        if csr is not None:
            return sq.scqr3_factor_oblique_csr(X, csr, **kw)
        if cfg.oblique:
            return sq.scqr3_factor_oblique(X, d, e, **kw)
        return sq.scqr3_factor(X, **kw)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            res = step()
            assert res.status == 0, f"warm-up step failed with status {res.status}"
    stream.synchronize()
    if multi:
        dist.barrier()
    torch.cuda.synchronize()

    clocks = Clocks(local if world > 1 else 0)
    sq.launch_count(reset=True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    clocks.start()
    time.sleep(0.3)
    # timed region: the default call path (single GPU: the cached CUDA-graph pass loop; with a
    # communicator: the host-driven pass loop), no profiling events
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for _ in range(args.steps):
            res = step()
        ev1.record(stream)
    stream.synchronize()
    clk = clocks.stop()
    launches = sq.launch_count()
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = flops_3pass(m, n) / (ms * 1e-3) / 1e12
    passes = res.passes
    actual = passes * m * (2.0 * n * n + n) / (ms * 1e-3) / 1e12

    # ---- profiled replay of the same steps right after the timed region: CUDA events recorded
    # by the library on `stream` around every launch (host-driven pass loop) give each kernel's
    # duration; its step time is reported beside the headline
    with torch.cuda.stream(stream):
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        for _ in range(args.steps):
            step(with_prof=True)
        p1.record(stream)
    stream.synchronize()
    ms_prof = p0.elapsed_time(p1) / args.steps

    # ---- quality of the last factorisation (outside the timed regions): orthogonality and
    # residual with the compensated metrics of tests/gpu_metrics.py (pinned to the oracle's Dot2
    # metrics); the north star asks for both <= 10 n u on every config
    quality = None
    if world == 1:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import gpu_metrics  # noqa: E402

        t_q = time.perf_counter()
        if csr is not None:
            orth = None  # (the CSR metric's Q^T B Q check lives in the tests)
        elif cfg.oblique:
            orth = float(gpu_metrics.orth_F(Q, d, e))
        else:
            orth = float(gpu_metrics.orth_F(Q))
        resid = float(gpu_metrics.resid_F(X, Q, R))
        quality = {"orth_F": orth, "resid_F": resid, "ten_n_u": 10 * n * 2.0 ** -53,
                   "metric": ("||Q^T B Q - I||_F" if cfg.oblique else "||Q^T Q - I||_F") + " and ||X - QR||_F / ||X||_F, "
                             "compensated (tests/gpu_metrics.py)", "seconds": time.perf_counter() - t_q}

    # ---- per-kernel device time measured live during the timed steps (events on `stream`)
    peaks = load_json(FP64_PEAKS) or {}
    peak = peaks.get("roofline_fp64_peak_tflops", 37.1)
    kern = {}
    # n <= 64, standard inner product: every TRSM launch but a step's last also accumulates the
    # next pass's Gram (trsm_kernel<..., GRAM>), so its algorithmic work carries that Gram too
    fused = (not cfg.oblique) and n <= 64 and os.environ.get("SCQR3_FUSE_TG", "1") != "0"
    fl_trsm = mloc * float(n) * n
    if fused and passes > 0:
        fl_trsm += (passes - 1) / passes * mloc * n * (n + 1.0)
    # the oblique Gram kernel also forms the plain Gram (upper tiles) for the norm estimate (D4)
    fl_gram = mloc * n * (n + 1.0) * (2 if cfg.oblique else 1)
    for name, msum, cnt, fl in (("gram", prof.gram_ms, prof.gram_launches, fl_gram),
                                ("trsm", prof.trsm_ms, prof.trsm_launches, fl_trsm),
                                ("chol", prof.chol_ms, prof.chol_launches, None),
                                ("reduce", prof.reduce_ms, prof.reduce_launches, None),
                                ("comm", prof.comm_ms, prof.comm_calls, None)):
        if cnt:
            avg = msum / cnt
            kern[name] = {"avg_ms": avg, "launches": int(cnt), "share_of_step": msum / (ms_prof * args.steps)}
            if fl:
                kern[name]["tflops"] = fl / (avg * 1e-3) / 1e12
                kern[name]["frac_of_peak"] = kern[name]["tflops"] / peak
    dom = max(("gram", "trsm"), key=lambda k: kern.get(k, {}).get("avg_ms", 0) * kern.get(k, {}).get("launches", 0))
    traffic_tab = load_json(NCU_TRAFFIC) or {}
    tr = traffic_tab.get(f"{args.config}:{dom}")
    roofline = {"bound": "tensor", "achieved": kern[dom]["tflops"], "peak": peak, "unit": "TFLOP/s",
                "frac": kern[dom]["tflops"] / peak, "traffic": tr.get("bytes_per_launch") if tr else None,
                "kernel": f"{dom}_kernel (FP64 DMMA)" + (" + fused next-pass Gram" if dom == "trsm" and fused else "")
                          + (" + trsm_wide_kernel (block-column launches, one timed unit)" if dom == "trsm" and n > 128
                             else "")
                          + (" (B-Gram + plain Gram)" if dom == "gram" and cfg.oblique else ""),
                "peak_source": "measured FP64 DMMA loop on this pool's B200 (profiles/fp64_peaks.json); "
                               "MEASURED_PEAKS.json has no fp64 entry",
                "algorithmic_flops_per_launch": fl_gram if dom == "gram" else fl_trsm}
    step_roof_ms, step_model = executed_roofline_ms(cfg, mloc, n, passes, peak, fused,
                                                    nnz=(int(csr.vals.numel()) if csr is not None else 0))

    # ---- end to end through the C ABI with host buffers (H2D of X, D2H of Q and R inside)
    e2e = None
    e2e_note = None
    want_e2e = not args.no_e2e and not cfg.oblique
    if want_e2e:
        # pinned host X and Q of every rank on this node (C4: 164 GB) must fit in host memory;
        # rank 0 decides for all ranks so that they stay in step
        need = 16.0 * m * n
        ok = torch.tensor([1.0 if need < 0.5 * host_mem_available() else 0.0], dtype=torch.float64, device=dev)
        if multi:
            dist.broadcast(ok, src=0)
        if ok.item() == 0.0:
            want_e2e = False
            e2e_note = (f"e2e skipped: pinned host X and Q need {need / 1e9:.0f} GB, more than half of the "
                        f"host's available memory ({host_mem_available() / 1e9:.0f} GB)")
    if want_e2e:
        Xh = torch.empty((n, mloc), dtype=torch.float64, pin_memory=True).t()
        Xh.copy_(X)
        Qh = torch.empty((n, mloc), dtype=torch.float64, pin_memory=True).t()
        Rh = torch.empty((n, n), dtype=torch.float64, pin_memory=True).t()
        wsh = sq.workspace(mloc, n, host_io=True, device=dev)
        del ws
        torch.cuda.empty_cache()
        with torch.cuda.stream(stream):
            sq.scqr3_factor_host(Xh, Q=Qh, R=Rh, ws=wsh, comm=comm, m_global=m, stream=stream)  # warm-up
            if multi:
                dist.barrier()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(args.e2e_steps):
                rh = sq.scqr3_factor_host(Xh, Q=Qh, R=Rh, ws=wsh, comm=comm, m_global=m, stream=stream)
            a1.record(stream)
        stream.synchronize()
        ems1 = a0.elapsed_time(a1) / args.e2e_steps
        # streaming: scqr3_factor_host_batch over e2e_steps matrices (each uploaded, factored and
        # downloaded; the uploads / downloads of neighbouring matrices overlap the factorisation)
        del wsh
        torch.cuda.empty_cache()
        ebatch = max(args.e2e_steps, 8)
        try:
            wsb = torch.empty(sq._abi.lib().scqr3_host_batch_workspace_size(mloc, n), dtype=torch.uint8, device=dev)
        except torch.cuda.OutOfMemoryError:  # three staging buffers do not fit: one matrix per call
            wsb = None
        okb = torch.tensor([0.0 if wsb is None else 1.0], dtype=torch.float64, device=dev)
        if multi:
            dist.all_reduce(okb, op=dist.ReduceOp.MIN)  # the same choice on every rank
        if okb.item() == 0.0:
            wsb = None
    if want_e2e and wsb is None:
        e2e = {"value": flops_3pass(m, n) / (ems1 * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": 8 * mloc * n, "d2h_bytes_per_step": 8 * mloc * n + 8 * n * n,
               "ms_per_step": ems1, "status": rh.status,
               "api": "scqr3_factor_host (pinned host X in, pinned host Q and R out)"}
    elif want_e2e:
        with torch.cuda.stream(stream):
            sq.scqr3_factor_host_batch([Xh] * 2, [Qh] * 2, [Rh] * 2, ws=wsb, comm=comm, m_global=m,
                                       stream=stream)  # warm-up (graph captures of the staging buffers)
            if multi:
                dist.barrier()
            a0.record(stream)
            sts = sq.scqr3_factor_host_batch([Xh] * ebatch, [Qh] * ebatch, [Rh] * ebatch, ws=wsb, comm=comm,
                                             m_global=m, stream=stream)
            a1.record(stream)
        stream.synchronize()
        ems = a0.elapsed_time(a1) / ebatch
        te = torch.tensor([ems, ems1], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ems, ems1 = float(te[0].item()), float(te[1].item())
        del wsb
        e2e = {"value": flops_3pass(m, n) / (ems * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": 8 * mloc * n, "d2h_bytes_per_step": 8 * mloc * n + 8 * n * n,
               "ms_per_step": ems, "status": max(sts), "matrices": ebatch,
               "api": "scqr3_factor_host_batch (pinned host X in, pinned host Q and R out; the next matrix's "
                      "upload and the previous one's download overlap each factorisation)",
               "single_call": {"value": flops_3pass(m, n) / (ems1 * 1e-3) / 1e12, "ms_per_step": ems1,
                               "status": rh.status, "api": "scqr3_factor_host (one matrix per call)"}}

    # ---- CPU oracle baseline on a bounded sample of the same X (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle

        rows = args.cpu_rows or max(n, int(1e7 * (128 / n) ** 2))
        rows = min(rows, mloc)
        okw = {}
        if csr is not None:
            _, Bs, rows = synth.config_metric(cfg, rows)
            okw = dict(csr=Bs)
        elif cfg.oblique:
            okw = dict(d=d[:rows].cpu().numpy(), e=e[:rows].cpu().numpy())
        Xs = X[:rows].cpu().numpy()
        t0 = time.perf_counter()
        ro = oracle.scqr3(Xs, **okw)
        tc = time.perf_counter() - t0
        cpu = {"value": flops_3pass(rows, n) / tc / 1e12, "unit": "TFLOP/s", "cores": oracle.num_threads(),
               "kind": "oracle", "seconds": tc, "passes": ro.passes, "status": ro.status,
               "tflops_actual_passes": ro.passes * rows * (2.0 * n * n + n) / tc / 1e12,
               "cpu_model": cpu_model(),
               "sample": f"first {rows} of {m} rows of the same device-generated X ({args.config}), one factorisation"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: X fp64 m={m} n={n} kappa2={cfg.kappa:g} "
                                   f"({cfg.spectrum} sigma, U,V Householder of N(0,1)), seed 0",
                       "m": m, "n": n, "kappa": cfg.kappa, "passes": passes,
                       "shifted": [t["shifted"] for t in res.trace], "parallelism": f"row-block x{world}",
                       "l2": f"no flush: X and Q ({8 * mloc * n / 1e9:.2f} GB each per GPU) >> 126 MB L2"},
            "roofline": roofline,
            "roofline_step": {"ms": step_roof_ms, "frac": step_roof_ms / ms, "passes": passes,
                              "model": step_model},
            "ms_per_step_profiled": ms_prof,
            "tflops_actual_passes": actual,
            "kernels": kern,
            "cpu_baseline": cpu,
            "e2e": e2e,
            **({"e2e_note": e2e_note} if e2e_note else {}),
            "quality": quality,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.destroy()
    if multi:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
