"""Per-call latency of scqr3_factor (no profiling, so single-GPU calls take the CUDA-graph pass
loop unless SCQR3_GRAPH=0): python tools/latency.py [config] [reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1809_11085_b200 as sq  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "PR1"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
X = synth.randsvd_torch(cfg.m, cfg.n, cfg.kappa, seed=0, spectrum=cfg.spectrum)
Q = sq.colmajor_empty(cfg.m, cfg.n)
R = torch.empty((cfg.n, cfg.n), dtype=torch.float64, device="cuda").t()
ws = sq.workspace(cfg.m, cfg.n)
for _ in range(5):
    r = sq.scqr3_factor(X, Q=Q, R=R, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
for _ in range(reps):
    r = sq.scqr3_factor(X, Q=Q, R=R, ws=ws)
e1.record()
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"{cfg.name} m={cfg.m} n={cfg.n}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us/call (device), "
      f"{(t1 - t0) / reps * 1e6:.1f} us/call (host wall), passes={r.passes} status={r.status} "
      f"graph={'off' if os.environ.get('SCQR3_GRAPH') == '0' else 'on'}")
