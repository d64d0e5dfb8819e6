"""Full-size accuracy metrics computed on the GPU with library GEMMs (torch / cuBLAS) --
TEST INFRASTRUCTURE, independent of libscqr3's kernels.

At m = 1e7 a plain fp64 Gram of Q has rounding error comparable to the 10*n*u target, so the
orthogonality is accumulated from small row chunks (4096 rows: per-chunk GEMM error ~ chunk*u
relative to a chunk's O(chunk/m) contribution) summed in double-double (TwoSum) -- the same
compensated-accumulation idea as the oracle's Dot2 metrics."""
import torch


def _two_sum(s, c, x):
    t = s + x
    bp = t - s
    e = (s - (t - bp)) + (x - bp)
    return t, c + e


def orth_F(Q, d=None, e=None, chunk=4096, Y=None):
    """||Q^T Q - I||_F (or ||Q^T B Q - I||_F for tridiagonal B = (d, e), or for any B with
    Y = B Q given) in compensated fp64."""
    m, n = Q.shape
    s = torch.zeros((n, n), dtype=torch.float64, device=Q.device)
    c = torch.zeros_like(s)
    for r0 in range(0, m, chunk):
        r1 = min(m, r0 + chunk)
        Qc = Q[r0:r1]
        if Y is not None:
            Yc = Y[r0:r1]
        elif d is None:
            Yc = Qc
        else:  # rows r0..r1-1 of B Q: d_i q_i + e_{i-1} q_{i-1} + e_i q_{i+1}
            Yc = d[r0:r1, None] * Qc
            i0 = max(r0, 1)
            Yc[i0 - r0:] += e[i0 - 1:r1 - 1, None] * Q[i0 - 1:r1 - 1]
            i1 = min(r1, m - 1)
            Yc[:i1 - r0] += e[r0:i1, None] * Q[r0 + 1:i1 + 1]
        s, c = _two_sum(s, c, Qc.T @ Yc)
    G = s + c
    G.diagonal().sub_(1.0)
    return float(torch.linalg.norm(G))


def resid_F(X, Q, R, chunk=1 << 20):
    """||X - Q R||_F / ||X||_F (chunked cuBLAS products)."""
    m, n = X.shape
    num = torch.zeros((), dtype=torch.float64, device=X.device)
    den = torch.zeros((), dtype=torch.float64, device=X.device)
    Ru = torch.triu(R)
    for r0 in range(0, m, chunk):
        r1 = min(m, r0 + chunk)
        D = X[r0:r1] - Q[r0:r1] @ Ru
        num += (D * D).sum()
        den += (X[r0:r1] * X[r0:r1]).sum()
    return float(torch.sqrt(num / den))
