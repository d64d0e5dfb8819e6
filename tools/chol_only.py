"""Repeated kernel-level Cholesky calls (scqr3_cholesky) for ncu captures of chol_kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1809_11085_b200 as sq  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
A = torch.randn(4 * n, n, dtype=torch.float64, device="cuda")
A = (A.T @ A).contiguous()
for _ in range(5):
    R = sq.scqr3_cholesky(A)
torch.cuda.synchronize()
print("ok", type(R))
