"""Seeded synthetic inputs shaped like the paper's workloads (shared by tests, bench, smoke).

This module holds NONE of the method's arithmetic (no Gram, no Cholesky, no triangular
solve, no shift): it only draws random numbers and builds the paper's test matrices
("X := U Sigma V^T ... essentially MATLAB's randsvd"), plus the
BASELINE.json tridiagonal SPD metric B.  Both the oracle and the CUDA path consume what
it returns; neither is imported here.

Recipes:
  * U (m x n) and V (n x n): Householder QR (LAPACK geqrf/orgqr via numpy on the host; on the
    device a Householder TSQR over fixed 2^20-row chunks, each drawn from its own seeded
    generator, so a rank can generate just its own rows -- reading D17) of i.i.d. N(0,1)
    matrices, columns sign-normalised so diag(R) > 0.
  * sigma geometric: sigma_i = kappa^{-(i-1)/(n-1)}, i = 1..n (||X||_2 = 1, kappa_2 = kappa).
  * sigma "cluster" (BASELINE config 4, reading D15): sigma_1 = 1, sigma_2..sigma_{n-8}
    log-uniform in [1e-6, 1] sorted descending, the last 8 equal to 1/kappa (= 1e-14).
  * B: d_i log-uniform in [1, 1e4], e_i = -0.45 sqrt(d_i d_{i+1}) (B = D^1/2 T D^1/2, T SPD).
Host streams: numpy PCG64 default_rng([seed, tag]); device streams: torch CUDA generator
seeded with seed (a different stream, stated in DESIGN.md; each arm always compares
like with like because the oracle receives the very array the GPU factorised).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TAG_U, TAG_V, TAG_SIGMA, TAG_B = 1, 2, 3, 4


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    kappa: float
    spectrum: str = "geometric"   # or "cluster"
    oblique: bool = False
    gpus: tuple = (1,)
    metric: str = "tridiag"       # oblique metric: "tridiag" (BASELINE config 5) or "laplacian"
    grid_nx: int = 1000           # laplacian: grid width (m = grid_nx * ny)


# BASELINE.json "configs" (index 0..4)
CONFIGS = {
    "PR1": Config("PR1", 2000, 16, 1e12),
    "C2": Config("C2", 1_000_000, 64, 1e15),
    "C3": Config("C3", 10_000_000, 128, 1e10, gpus=(1, 2, 4, 8)),
    "C4": Config("C4", 40_000_000, 256, 1e14, spectrum="cluster", gpus=(4, 8)),
    "C5": Config("C5", 2_000_000, 64, 1e12, oblique=True, gpus=(1, 8)),
    # C5 with a general sparse SPD metric in CSR (stand-in for the paper's
    # sparse matrices): weighted 5-point Laplacian on a 1000 x 2000 grid
    "C5L": Config("C5L", 2_000_000, 64, 1e12, oblique=True, gpus=(1, 8), metric="laplacian"),
}


def config_metric(cfg: Config, rows: int):
    """The oblique metric of a config restricted to its first `rows` rows (a principal
    submatrix): tridiagonal bands (d, e), or the weighted Laplacian of the first rows // nx
    grid lines as CSR.  Returns (kind, data, rows_used)."""
    if cfg.metric == "laplacian":
        ny = max(1, rows // cfg.grid_nx)
        return "csr", laplacian2d(cfg.grid_nx, ny, seed=0, wmax=1e4), cfg.grid_nx * ny
    return "tridiag", tridiag_b(rows, seed=0), rows


def sigma(n: int, kappa: float, spectrum: str = "geometric", seed: int = 0) -> np.ndarray:
    if n == 1:
        return np.ones(1)
    if spectrum == "geometric":
        i = np.arange(n, dtype=np.float64)
        return kappa ** (-i / (n - 1))
    if spectrum == "cluster":
        rng = np.random.default_rng([seed, TAG_SIGMA])
        k = min(8, n - 1)
        mid = np.sort(10.0 ** rng.uniform(-6.0, 0.0, size=n - 1 - k))[::-1]
        return np.concatenate([[1.0], mid, np.full(k, 1.0 / kappa)])
    raise ValueError(spectrum)


def _signed_qr(G: np.ndarray) -> np.ndarray:
    Q, R = np.linalg.qr(G, mode="reduced")
    s = np.sign(np.diag(R))
    s[s == 0] = 1.0
    return Q * s


def randsvd(m: int, n: int, kappa: float, seed: int = 0, spectrum: str = "geometric") -> np.ndarray:
    """X = U diag(sigma) V^T as an m x n column-major (Fortran) float64 array."""
    rng_u = np.random.default_rng([seed, TAG_U])
    rng_v = np.random.default_rng([seed, TAG_V])
    U = _signed_qr(rng_u.standard_normal((m, n)))
    V = _signed_qr(rng_v.standard_normal((n, n)))
    s = sigma(n, kappa, spectrum, seed)
    X = (U * s) @ V.T
    return np.asfortranarray(X)


def _signed_zqr(G: np.ndarray) -> np.ndarray:
    """Thin unitary Q of a complex G with the phases normalised so diag(R) > 0 (unique)."""
    Q, R = np.linalg.qr(G, mode="reduced")
    d = np.diag(R)
    ph = np.where(np.abs(d) > 0, d / np.abs(d), 1.0)
    return Q * ph


def randsvd_complex(m: int, n: int, kappa: float, seed: int = 0, spectrum: str = "geometric") -> np.ndarray:
    """Complex X = U diag(sigma) V^H (P:1510-1521 recipe with unitary U, V from complex Gaussians;
    N4), column-major complex128."""
    rng_u = np.random.default_rng([seed, TAG_U, 1])
    rng_v = np.random.default_rng([seed, TAG_V, 1])
    U = _signed_zqr((rng_u.standard_normal((m, n)) + 1j * rng_u.standard_normal((m, n))) / np.sqrt(2))
    V = _signed_zqr((rng_v.standard_normal((n, n)) + 1j * rng_v.standard_normal((n, n))) / np.sqrt(2))
    s = sigma(n, kappa, spectrum, seed)
    return np.asfortranarray((U * s) @ V.conj().T)


def tridiag_b(m: int, seed: int = 0):
    """Bands (d, e) of the SPD tridiagonal metric of BASELINE config 5; e[m-1] = 0 (unused)."""
    rng = np.random.default_rng([seed, TAG_B])
    d = 10.0 ** rng.uniform(0.0, 4.0, size=m)
    e = np.zeros(m)
    e[:-1] = -0.45 * np.sqrt(d[:-1] * d[1:])
    return d, e


def tridiag_csr(d: np.ndarray, e: np.ndarray):
    """The tridiagonal metric (d, e) in CSR, each row's entries in the order (i, i-1, i+1)
    (the term order of the banded formula), so both forms describe the same operation."""
    m = d.size
    rp = np.zeros(m + 1, dtype=np.int64)
    ci, cv = [], []
    for i in range(m):
        ci.append(i); cv.append(d[i])
        if i > 0:
            ci.append(i - 1); cv.append(e[i - 1])
        if i + 1 < m:
            ci.append(i + 1); cv.append(e[i])
        rp[i + 1] = len(ci)
    return rp, np.asarray(ci, dtype=np.int32), np.asarray(cv, dtype=np.float64)


def laplacian2d(nx: int, ny: int, seed: int | None = None, wmax: float = 1.0):
    """5-point 2-D Laplacian on an nx x ny grid (Dirichlet), m = nx*ny rows in row-major grid
    order, as CSR (row_ptr int64, col_idx int32, vals float64) with each row's diagonal first,
    then the neighbours ascending -- the synthetic stand-in for the paper's sparse SPD B
    (not available).  With seed: D^1/2 L D^1/2, d_i log-uniform in
    [1, wmax] (still SPD)."""
    m = nx * ny
    i = np.arange(m)
    gx, gy = i % nx, i // nx
    w = np.ones(m) if seed is None else 10.0 ** np.random.default_rng([seed, TAG_B]).uniform(0.0, np.log10(wmax), m)
    sw = np.sqrt(w)
    nbr = [(gy > 0, -nx), (gx > 0, -1), (gx + 1 < nx, 1), (gy + 1 < ny, nx)]
    cnt = 1 + sum(ok.astype(np.int64) for ok, _ in nbr)
    rp = np.zeros(m + 1, dtype=np.int64)
    rp[1:] = np.cumsum(cnt)
    ci = np.empty(rp[-1], dtype=np.int32)
    cv = np.empty(rp[-1], dtype=np.float64)
    pos = rp[:-1].copy()
    ci[pos] = i
    cv[pos] = 4.0 * w
    pos += 1
    for ok, off in nbr:
        rows = i[ok]
        ci[pos[ok]] = rows + off
        cv[pos[ok]] = -sw[rows] * sw[rows + off]
        pos[ok] += 1
    return rp, ci, cv


def csr_rows(B, r0: int, r1: int):
    """Rows [r0, r1) of a CSR matrix with column indices made relative to r0 (a rank's shard;
    neighbours' rows appear as negative / >= r1-r0 indices, served by the halo)."""
    rp, ci, cv = B
    a, b = rp[r0], rp[r1]
    return rp[r0:r1 + 1] - a, (ci[a:b].astype(np.int64) - r0).astype(np.int32), cv[a:b].copy()


def random_rows(m: int, n: int, seed: int = 0) -> np.ndarray:
    """Plain i.i.d. N(0,1) column-major matrix (kernel-level tests)."""
    rng = np.random.default_rng([seed, 7])
    return np.asfortranarray(rng.standard_normal((m, n)))


# --------------------------------------------------------------------------- device side
CHUNK_ROWS = 1 << 20  # device generator: rows per seeded Gaussian chunk (independent of the GPU count)


def randsvd_torch(m: int, n: int, kappa: float, seed: int = 0, spectrum: str = "geometric",
                  device="cuda", ld: int | None = None):
    """Same recipe on the device; returns the whole (m, n) X with column-major strides (1, ld).
    (randsvd_torch_rows with one rank.)"""
    return randsvd_torch_rows(m, n, kappa, 0, m, seed=seed, spectrum=spectrum, device=device, ld=ld)


def randsvd_torch_rows(m: int, n: int, kappa: float, r0: int, r1: int, seed: int = 0, spectrum: str = "geometric",
                       device="cuda", ld: int | None = None, allreduce=None):
    """Rows [r0, r1) of X = U diag(sigma) V^T generated on the device without
    forming the other rows, so each rank of a multi-GPU run makes only its own block.

    U is the thin Q factor of an m x n N(0,1) matrix G, by Householder TSQR (reading D17): G's
    fixed 2^20-row chunks are drawn from generators seeded per chunk (seed, chunk), each chunk
    is QR-factorised (cuSOLVER), the chunks' R factors are stacked and QR-factorised again, and
    chunk c's rows of U are Q_c times block c of that second Q, signs normalised so the
    overall R has a positive diagonal.  The result does not depend on how the rows are split
    over ranks.  `allreduce(t)` sums a tensor over the ranks in place (None: one rank); each
    chunk's R is contributed by the rank holding the chunk's first row (others add zeros).
    Returns an (r1 - r0, n) view with strides (1, ld)."""
    import torch

    if not (0 <= r0 <= r1 <= m):
        raise ValueError("bad row range")
    mr = r1 - r0
    ld = ld or max(mr, 1)
    C = CHUNK_ROWS
    nch = (m + C - 1) // C
    mine = [c for c in range(nch) if c * C < r1 and min(m, (c + 1) * C) > r0] if mr > 0 else []

    def chunk_qr(c):
        g = torch.Generator(device=device)
        g.manual_seed((int(seed) * 1000003 + TAG_U) * 65537 + c)
        rows = min(m, (c + 1) * C) - c * C
        Gc = torch.randn((n, rows), generator=g, dtype=torch.float64, device=device).t()
        return torch.linalg.qr(Gc, mode="reduced")

    Rs = torch.zeros((nch, n, n), dtype=torch.float64, device=device)
    Qc = {}
    for c in mine:
        Qm, Rm = chunk_qr(c)
        Qc[c] = Qm
        if r0 <= c * C:  # this rank holds the chunk's first row: it contributes R_c
            Rs[c].copy_(Rm)
    if allreduce is not None:
        allreduce(Rs)
    Q2, R2 = torch.linalg.qr(Rs.reshape(nch * n, n), mode="reduced")
    sgn = torch.sign(torch.diagonal(R2))
    sgn[sgn == 0] = 1.0
    gv = torch.Generator(device=device)
    gv.manual_seed(int(seed) * 1000003 + TAG_V)
    Gv = torch.randn((n, n), generator=gv, dtype=torch.float64, device=device)
    Vq, Vr = torch.linalg.qr(Gv)
    Vq = Vq * torch.sign(torch.diagonal(Vr))
    s = torch.as_tensor(sigma(n, kappa, spectrum, seed), dtype=torch.float64, device=device)
    W = (sgn * s)[:, None] * Vq.t()                       # diag(sgn*sigma) V^T, n x n
    out = torch.empty((n, ld), dtype=torch.float64, device=device)
    X = out.t()[:mr]
    for c in mine:
        a, b = max(r0, c * C), min(r1, (c + 1) * C)
        Mc = Q2[c * n:(c + 1) * n] @ W                      # block c of the second Q, times diag(sigma) V^T
        X[a - r0:b - r0].copy_(Qc[c][a - c * C:b - c * C] @ Mc)
        del Qc[c]
    return X


def tridiag_b_torch(m: int, seed: int = 0, device="cuda"):
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 1000003 + TAG_B)
    d = 10.0 ** (torch.rand(m, generator=g, dtype=torch.float64, device=device) * 4.0)
    e = torch.zeros(m, dtype=torch.float64, device=device)
    e[:-1] = -0.45 * torch.sqrt(d[:-1] * d[1:])
    return d, e
