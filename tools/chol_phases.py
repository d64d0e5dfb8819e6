"""Phase timing of chol_kernel (clock64 stamps left in the workspace's status block)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_11085_b200 as sq  # noqa: E402
import synth  # noqa: E402

for n in (16, 64, 128, 256):
    m = 200000
    X = synth.randsvd_torch(m, n, 1e10, seed=0)
    ws = sq.workspace(m, n)
    for rep in range(2):
        r = sq.scqr3_factor(X, ws=ws, max_passes=int(os.environ.get("MAXP", "2")),
                            power_iters=int(os.environ.get("PITERS", "32")))
    st = ws[:160].cpu().numpy().view(np.int64)
    clk = st[56 // 8: 56 // 8 + 8]
    d = np.diff(clk[:6])
    print(f"n={n} passes={r.passes} (last pass) cycles: load={d[0]} dev={d[1]} norm={d[2]} "
          f"factor={d[3]} [a={clk[6]} b={clk[7]} c={d[3]-clk[6]-clk[7]}] outputs+status={d[4]}  "
          f"total={clk[5]-clk[0]} (~{(clk[5]-clk[0])/1.9e3:.1f} us)")
