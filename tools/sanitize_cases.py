"""Small factorisations covering every kernel family of libscqr3, for compute-sanitizer runs
(one tool per process):

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Cases (rows >= two persistent TRSM sweeps where the kernel is persistent):
  pr1       n=16 (PR1 shape; CUDA-graph pass loop)
  fused40   n=40: fused TRSM + next-pass Gram, bulk tensor stores of Q
  n128      n=128: register-resident TRSM, TMA Gram (m = 40,000 > 2 x 18,944 rows)
  n256      n=256: block-column TRSM (resident targets 16..31), whole-block Gram variant
  n300      n=300: resident launches for targets 32..40
  oblique   tridiagonal metric, n=64 (Y kernel, dual Gram)
  csr       2-D Laplacian metric in CSR, n=32
  complex   complex X, n=24 (split matrix, zchol)
  loopback  P=2 loopback ranks, standard + tridiagonal metric
Each case checks status 0 (the numerics are covered by the parity tests)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_11085_b200 as sq  # noqa: E402
import synth  # noqa: E402
from paper_1809_11085_b200.dist import row_block, run_ranks  # noqa: E402


def dev(X):
    return sq.to_colmajor(torch.from_numpy(np.asfortranarray(X)), device="cuda")


def std(m, n, kappa):
    r = sq.scqr3_factor(dev(synth.randsvd(m, n, kappa, seed=1)))
    assert r.status == 0, r.status
    return r.passes


CASES = {
    "pr1": lambda: std(2000, 16, 1e12),
    "fused40": lambda: std(40_000, 40, 1e9),
    "n128": lambda: std(40_000, 128, 1e10),
    "n256": lambda: std(40_000, 256, 1e8),
    "n300": lambda: std(40_000, 300, 1e8),
}


def oblique():
    m, n = 40_000, 64
    X = synth.randsvd(m, n, 1e10, seed=2)
    d, e = synth.tridiag_b(m, seed=2)
    r = sq.scqr3_factor_oblique(dev(X), torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda())
    assert r.status == 0
    return r.passes


def csr():
    nx, ny, n = 100, 200, 32
    B = synth.laplacian2d(nx, ny, seed=0, wmax=1e3)
    X = synth.randsvd(nx * ny, n, 1e8, seed=3)
    r = sq.scqr3_factor_oblique_csr(dev(X), sq.CsrMetric(*B))
    assert r.status == 0
    return r.passes


def complex_():
    Z = synth.randsvd_complex(20_000, 24, 1e9, seed=4)
    Zd = torch.from_numpy(np.asfortranarray(Z)).cuda().t().contiguous().t()
    r = sq.scqr3_factor_complex(Zd)
    assert r.status == 0
    return r.passes


def loopback():
    P, m, n = 2, 40_000, 32
    X = synth.randsvd(m, n, 1e10, seed=5)
    d, e = synth.tridiag_b(m, seed=5)
    comms = sq.Comm.loopback(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    parts = [row_block(m, r, P) for r in range(P)]
    Xs = [dev(X[a:b]) for a, b in parts]
    ds = [torch.from_numpy(d[a:b].copy()).cuda() for a, b in parts]
    es = [torch.from_numpy(e[a:b].copy()).cuda() for a, b in parts]
    torch.cuda.synchronize()
    res = run_ranks([lambda r=r: sq.scqr3_factor(Xs[r], comm=comms[r], stream=streams[r]) for r in range(P)])
    res += run_ranks([lambda r=r: sq.scqr3_factor_oblique(Xs[r], ds[r], es[r], comm=comms[r], stream=streams[r])
                      for r in range(P)])
    for c in comms:
        c.destroy()
    assert all(x.status == 0 for x in res)
    return res[0].passes


CASES.update({"oblique": oblique, "csr": csr, "complex": complex_, "loopback": loopback})

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for name in names:
        passes = CASES[name]()
        torch.cuda.synchronize()
        print(f"case {name}: ok ({passes} passes)", flush=True)
