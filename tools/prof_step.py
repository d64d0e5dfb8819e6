"""One (or a few) shifted CholeskyQR3 factorisations of a C3-shaped matrix, for ncu captures.

  python tools/prof_step.py [--m 2000000] [--n 128] [--reps 2] [--oblique]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1809_11085_b200 as sq  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=2_000_000)
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--kappa", type=float, default=1e10)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--oblique", action="store_true")
a = ap.parse_args()

X = synth.randsvd_torch(a.m, a.n, a.kappa, seed=0)
ws = sq.workspace(a.m, a.n, oblique=a.oblique)
Q = sq.colmajor_empty(a.m, a.n)
if a.oblique:
    d, e = synth.tridiag_b_torch(a.m, seed=0)
for _ in range(a.reps):
    if a.oblique:
        r = sq.scqr3_factor_oblique(X, d, e, Q=Q, ws=ws)
    else:
        r = sq.scqr3_factor(X, Q=Q, ws=ws)
torch.cuda.synchronize()
print("status", r.status, "passes", r.passes)
