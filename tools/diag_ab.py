"""A/B of the TRSM's diagonal-block modes (reading D24) through scqr3_factor on the device.

  python tools/diag_ab.py [config ...]      (configs: C3 C2 C5 N256 N192 N96; default C3 C2)
For each config: ms per factorisation (graph path, best of 5) and the profiled TRSM ms per
launch with trsm_diag = SUBST and AUTO, the passes, max|dR| / max|R| between the two, and both
results' orthogonality / residual (tests/gpu_metrics.py, Dot2)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402
import paper_1809_11085_b200 as sq  # noqa: E402
from paper_1809_11085_b200 import _abi  # noqa: E402
import synth  # noqa: E402
import gpu_metrics  # noqa: E402

CFG = {"C3": (10_000_000, 128, 1e10, "geometric"), "C2": (1_000_000, 64, 1e15, "geometric"),
       "C5": (2_000_000, 64, 1e12, "geometric"), "N256": (5_000_000, 256, 1e14, "cluster"),
       "N192": (4_000_000, 192, 1e12, "geometric"), "N96": (4_000_000, 96, 1e12, "geometric"),
       "C3s": (2_000_000, 128, 1e10, "geometric"), "N512": (2_000_000, 512, 1e12, "geometric"),
       "N300": (2_000_000, 300, 1e12, "geometric")}
names = sys.argv[1:] or ["C3", "C2"]
u = 2.0 ** -53
for name in names:
    m, n, kap, spec = CFG[name]
    X = synth.randsvd_torch(m, n, kap, seed=0, spectrum=spec)
    obl = name == "C5"
    if obl:
        d, e = synth.tridiag_b_torch(m, seed=0)
    ws = sq.workspace(m, n, oblique=obl) if obl else sq.workspace(m, n)
    Q = sq.colmajor_empty(m, n)
    out = {}
    for mode, label in ((sq.TRSM_DIAG_SUBST, "subst"), (sq.TRSM_DIAG_AUTO, "auto")):
        def run(**kw):
            if obl:
                return sq.scqr3_factor_oblique(X, d, e, Q=Q, ws=ws, trsm_diag=mode, **kw)
            return sq.scqr3_factor(X, Q=Q, ws=ws, trsm_diag=mode, **kw)
        for _ in range(2):
            r = run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(5):
            e0.record()
            r = run()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        prof = _abi.Prof()
        run(prof=prof)
        torch.cuda.synchronize()
        R = r.R.clone()
        if obl:
            orth = gpu_metrics.orth_F(Q, d, e)
        else:
            orth = gpu_metrics.orth_F(Q)
        res = gpu_metrics.resid_F(X, Q, R)
        out[label] = R
        print(f"{name} m={m} n={n} {label:5s}: {min(ts):8.3f} ms  passes {r.passes}  trsm {prof.trsm_ms / max(prof.trsm_launches, 1):.3f} ms/pass"
              f"  gram {prof.gram_ms / max(prof.gram_launches, 1):.3f}  chol {prof.chol_ms / max(prof.chol_launches, 1) * 1e3:.1f} us"
              f"  orth {orth:.2e} resid {res:.2e} (10nu {10 * n * u:.2e}) status {r.status}", flush=True)
    dR = (out["subst"] - out["auto"]).abs().max().item() / out["subst"].abs().max().item()
    print(f"{name}: max|R_subst - R_auto| / max|R| = {dR:.2e}", flush=True)
    del X, Q, ws
    torch.cuda.empty_cache()
