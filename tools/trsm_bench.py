"""Time the TRSM and Gram kernels alone (kernel-level C-ABI calls) on a C3-shaped matrix."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1809_11085_b200 as sq  # noqa: E402
from paper_1809_11085_b200 import _abi  # noqa: E402
m = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
X = sq.colmajor_empty(m, n)
X.copy_(torch.randn(n, m, dtype=torch.float64, device="cuda").t())
R = torch.triu(torch.randn(n, n, dtype=torch.float64, device="cuda")) + 4 * torch.eye(n, device="cuda", dtype=torch.float64)
Q = sq.colmajor_empty(m, n)
ws = sq.workspace(m, n)
for _ in range(2):
    sq.scqr3_trsm(X, R, Q=Q, ws=ws)
    sq.scqr3_gram(X, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, fl in (("trsm", lambda: sq.scqr3_trsm(X, R, Q=Q, ws=ws), m * n * n),
                     ("gram", lambda: sq.scqr3_gram(X, ws=ws), m * n * (n + 1))):
    ts = []
    for _ in range(5):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    t = min(ts)
    print(f"{name} m={m} n={n}: {t:.3f} ms  {fl / t / 1e9:.2f} TF/s ({fl / t / 1e9 / 37.1 * 100:.1f}% of 37.1)")
