"""Complex shifted CholeskyQR3 timing: python tools/complex_bench.py [m] [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1809_11085_b200 as sq  # noqa: E402
from paper_1809_11085_b200 import _abi  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
X = sq.colmajor_empty_complex(m, n)
X.copy_(torch.randn(n, m, dtype=torch.complex128, device="cuda").t())
Q = sq.colmajor_empty_complex(m, n)
R = torch.empty((n, n), dtype=torch.complex128, device="cuda").t()
ws = torch.empty(_abi.lib().scqr3_workspace_size_complex(m, n), dtype=torch.uint8, device="cuda")
prof = _abi.Prof()
for _ in range(2):
    r = sq.scqr3_factor_complex(X, Q=Q, R=R, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    r = sq.scqr3_factor_complex(X, Q=Q, R=R, ws=ws, prof=prof)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
fl = r.passes * 2 * 4 * m * n * n  # executed passes x (Gram + TRSM), complex = 4 real multiply-adds
print(f"complex m={m} n={n}: {ms:.3f} ms, {fl / ms / 1e9:.2f} TF/s real-equivalent (executed passes), passes={r.passes} "
      f"gram {prof.gram_ms / max(prof.gram_launches, 1):.3f} ms trsm {prof.trsm_ms / max(prof.trsm_launches, 1):.3f} ms "
      f"chol {prof.chol_ms / max(prof.chol_launches, 1):.3f} ms")
