"""Kernel-level oblique Gram timing (tridiagonal B): python tools/gram_oblique_bench.py [m] [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1809_11085_b200 as sq  # noqa: E402
import synth  # noqa: E402
m = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
X = sq.colmajor_empty(m, n)
X.copy_(torch.randn(n, m, dtype=torch.float64, device="cuda").t())
d, e = synth.tridiag_b_torch(m)
ws = sq.workspace(m, n, oblique=True)
for _ in range(2):
    sq.scqr3_gram_oblique(X, d, e, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    sq.scqr3_gram_oblique(X, d, e, ws=ws)
e1.record()
torch.cuda.synchronize()
print(f"oblique gram m={m} n={n}: {e0.elapsed_time(e1) / 5:.3f} ms per call (Y + Gram + reduce)")
