"""Time the TRSM and Gram kernels alone (kernel-level C-ABI calls) on a C3-shaped matrix.

  python tools/trsm_bench.py [m] [n] [--only trsm] [--diag auto|subst|inverse]   (SCQR3_LIB selects a library build)
Prints the best of 5 timings per kernel and a hash of the TRSM output's first rows (A/B builds
that only reorder independent work must produce identical bits)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1809_11085_b200 as sq  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
diag = sys.argv[sys.argv.index("--diag") + 1] if "--diag" in sys.argv else "auto"  # reading D24
if only:
    args = [a for a in args if a != only]
args = [a for a in args if a != diag]
DIAG = {"auto": sq.TRSM_DIAG_AUTO, "subst": sq.TRSM_DIAG_SUBST, "inverse": sq.TRSM_DIAG_INVERSE}[diag]
m = int(args[0]) if len(args) > 0 else 10_000_000
n = int(args[1]) if len(args) > 1 else 128
g = torch.Generator(device="cuda")
g.manual_seed(1)
X = sq.colmajor_empty(m, n)
X.copy_(torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g).t())
R = torch.triu(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)) + 4 * torch.eye(
    n, device="cuda", dtype=torch.float64)
Q = sq.colmajor_empty(m, n)
ws = sq.workspace(m, n)
for _ in range(2):
    sq.scqr3_trsm(X, R, Q=Q, ws=ws, trsm_diag=DIAG)
    if only != "trsm":
        sq.scqr3_gram(X, ws=ws)
torch.cuda.synchronize()
h = hashlib.sha1(Q[:200_000].cpu().numpy().tobytes()).hexdigest()[:12]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, fl in (("trsm", lambda: sq.scqr3_trsm(X, R, Q=Q, ws=ws, trsm_diag=DIAG), m * n * n),
                     ("gram", lambda: sq.scqr3_gram(X, ws=ws), m * n * (n + 1))):
    if only and name != only:
        continue
    ts = []
    for _ in range(5):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    t = min(ts)
    print(f"{name} m={m} n={n}: {t:.3f} ms  {fl / t / 1e9:.2f} TF/s ({fl / t / 1e9 / 37.1 * 100:.1f}% of 37.1)"
          + (f" Qhash={h}" if name == "trsm" else ""))
