"""Y = BQ + oblique Gram time per call (kernel-level scqr3_gram_oblique_csr, CUDA events) for banded SPD metrics of
growing density: 5, 9, 13, 17 and 25 nonzeros per row (offsets 0, +-1, +-nx, ... on a 1000-wide
grid), m = 2e6, n = 64.  Run once per kernel: SCQR3_CSR_Y=0 (round-1 kernel) / 1 (tile kernel;
tiles with more than 12 nonzeros per row read ci / cv from global memory)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_11085_b200 as sq  # noqa: E402

m, n, nx = 2_000_000, 64, 1000
X = sq.to_colmajor(torch.randn(m, n, dtype=torch.float64, device="cuda"))
sets = {5: [1, nx], 9: [1, nx, nx - 1, nx + 1], 13: [1, 2, nx, 2 * nx, nx - 1, nx + 1],
        17: [1, 2, nx, 2 * nx, nx - 1, nx + 1, nx - 2, nx + 2],
        25: [1, 2, 3, nx, 2 * nx, 3 * nx, nx - 1, nx + 1, nx - 2, nx + 2, 2 * nx - 1, 2 * nx + 1]}
for k, offs in sets.items():
    offs = sorted([-o for o in offs] + offs)
    i = np.arange(m)
    cols = [i] + [i + o for o in offs]           # the diagonal first, then the bands ascending
    ok = [np.ones(m, bool)] + [(c >= 0) & (c < m) for c in cols[1:]]
    cnt = sum(o.astype(np.int64) for o in ok)
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(cnt)
    ci = np.empty(rp[-1], np.int32)
    cv = np.empty(rp[-1])
    pos = rp[:-1].copy()
    for c, o, v in zip(cols, ok, [float(len(offs) + 1)] + [-1.0] * len(offs)):
        ci[pos[o]] = c[o]
        cv[pos[o]] = v
        pos[o] += 1
    B = sq.CsrMetric(rp, ci, cv)
    ws = sq.workspace(m, n, device="cuda", csr_halo=0)
    for _ in range(3):
        sq.scqr3_gram_oblique_csr(X, B, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        sq.scqr3_gram_oblique_csr(X, B, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    print(f"SCQR3_CSR_Y={os.environ.get('SCQR3_CSR_Y', '1')} nnz/row={k} Y + dual Gram + reduce "
          f"{e0.elapsed_time(e1) / reps:.4f} ms per call (the Gram part is ~0.59 ms in both)", flush=True)
    del B, ws
