"""Parity of the CUDA path (called through the C ABI via the thin binding) against the CPU oracle.

Tolerances:
  * Gram:    |A_gpu - A_orc| <= 2 gamma_m |X|^T|X| entrywise (both satisfy P:260-262's T1 bound)
  * oblique: |A_gpu - A_orc| <= 4 gamma_m (|X|^T |B| |X|) entrywise
  * Cholesky / TRSM: exact (bitwise) on integer cases; on floating cases within the T2 / T3
    backward-error bounds evaluated in extended precision
  * end to end (reading D14): max|R_gpu - R_orc| <= 1e-10 max|R_orc|; Q within 1e-10 max|Q| for
    kappa <= 1e6, within 10 kappa u max|Q| for kappa <= 1e8; orthogonality and residual <= 10 n u
    (north star) for both.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
gpu = pytest.mark.gpu
U = 2.0 ** -53

if torch.cuda.is_available():
    import paper_1809_11085_b200 as sq


def dev(X):
    return sq.to_colmajor(torch.from_numpy(np.asfortranarray(X)), device="cuda")


def host(T):
    return np.asfortranarray(T.detach().cpu().numpy())


def gamma(k):
    return k * U / (1 - k * U)


# ------------------------------------------------------------------ Gram
@gpu
@pytest.mark.parametrize("m,n", [(1, 1), (15, 3), (16, 16), (17, 8), (1000, 7), (4099, 33), (20001, 64),
                                 (5000, 100), (30011, 128), (3000, 200), (2500, 256),
                                 (1500, 300), (1200, 512)])
def test_gram_parity(m, n):
    X = synth.random_rows(m, n, seed=m + n)
    A = host(sq.scqr3_gram(dev(X)))
    Ao = oracle.gram(X)
    bound = 2 * gamma(m) * (np.abs(X).T @ np.abs(X))
    assert np.all(np.abs(A - Ao) <= bound + 1e-300)
    assert np.array_equal(A, A.T)


@gpu
@pytest.mark.parametrize("m,n,pad", [(32 * 1001, 64, 0), (32 * 3001, 128, 0), (32 * 777, 61, 6), (32 * 500, 124, 2),
                                     (32, 64, 0), (32 * 20000, 128, 4)])
def test_gram_parity_32row_stages(m, n, pad):
    """m % 32 == 0 and 8 ceil(n / 8) in {64, 128}: the Gram streams 32-row stages through the 3-D
    tensor map (two swizzled 128-B lines per column and box, gram.cu RB = 2); same T1 bound, an
    exact integer case bit for bit, and a leading dimension past m."""
    X = synth.random_rows(m, n, seed=m + n)
    Xd = sq.colmajor_empty(m, n, ld=m + pad) if pad else dev(X)
    if pad:
        Xd.copy_(torch.from_numpy(X))
    A = host(sq.scqr3_gram(Xd))
    bound = 2 * gamma(m) * (np.abs(X).T @ np.abs(X))
    assert np.all(np.abs(A - oracle.gram(X)) <= bound + 1e-300)
    Xi = np.random.default_rng(m).integers(-40, 41, size=(m, n)).astype(float)
    Ai = host(sq.scqr3_gram(dev(Xi)))
    assert np.array_equal(Ai, (Xi.astype(np.int64).T @ Xi.astype(np.int64)).astype(float))


@gpu
def test_gram_exact_integers_bitwise():
    rng = np.random.default_rng(5)
    X = rng.integers(-40, 41, size=(7777, 72)).astype(float)
    A = host(sq.scqr3_gram(dev(X)))
    assert np.array_equal(A, (X.astype(np.int64).T @ X.astype(np.int64)).astype(float))


@gpu
def test_gram_ld_padding_and_determinism():
    m, n = 12345, 40
    X = synth.random_rows(m, n, seed=2)
    Xd = sq.colmajor_empty(m, n, ld=m + 13)  # even ld > m
    Xd.copy_(torch.from_numpy(X))
    A1 = host(sq.scqr3_gram(Xd))
    A2 = host(sq.scqr3_gram(Xd))
    assert np.array_equal(A1, A2)
    bound = 2 * gamma(m) * (np.abs(X).T @ np.abs(X))
    assert np.all(np.abs(A1 - oracle.gram(X)) <= bound)


@gpu
@pytest.mark.parametrize("m,n", [(2, 1), (999, 16), (20000, 64), (3001, 128), (2500, 200), (1500, 300)])
def test_gram_oblique_parity(m, n):
    X = synth.random_rows(m, n, seed=n)
    d, e = synth.tridiag_b(m, seed=n)
    A, cs = sq.scqr3_gram_oblique(dev(X), torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda())
    Ao, cso = oracle.gram_oblique(X, d, e)
    B = np.abs(d)[:, None] * np.abs(X)
    B[1:] += np.abs(e[:-1])[:, None] * np.abs(X[:-1])
    B[:-1] += np.abs(e[:-1])[:, None] * np.abs(X[1:])
    bound = 4 * gamma(m + 2) * (np.abs(X).T @ B)
    assert np.all(np.abs(host(A) - Ao) <= bound)
    assert abs(cs.item() - cso.sum()) <= 4 * gamma(m * n) * cso.sum()


# ------------------------------------------------------------------ Cholesky
@gpu
@pytest.mark.parametrize("n", [1, 2, 9, 40, 128, 200, 256, 301, 512])
def test_cholesky_integer_exact(n):
    rng = np.random.default_rng(n)
    R = np.triu(rng.integers(-3, 4, size=(n, n))).astype(float)
    R[np.diag_indices(n)] = rng.integers(1, 6, size=n)
    A = R.T @ R
    Rg = sq.scqr3_cholesky(dev(A))
    assert np.array_equal(host(Rg), R)


@gpu
def test_cholesky_breakdown_matches_oracle():
    for A, piv in [(np.array([[1.0, 1.0], [1.0, 1.0]]), 2), (np.diag([1.0, 2.0, -1.0, 3.0]), 3)]:
        r = sq.scqr3_cholesky(dev(A))
        o = oracle.cholesky(A)
        assert r[0] == "breakdown" and r[1] == o.pivot == piv
    X = synth.randsvd(1000, 30, 1e12, seed=1)
    A = oracle.gram(X)
    assert sq.scqr3_cholesky(dev(A))[0] == "breakdown"
    s = oracle.shift(1000, 30, 1.0)
    Rg = host(sq.scqr3_cholesky(dev(A), s))
    Ro = oracle.cholesky(A, s)
    assert np.max(np.abs(Rg - Ro)) <= 1e-8 * np.max(np.abs(Ro))   # kappa(A+sI) ~ 1/alpha
    # T2 backward error of the GPU factor, evaluated in extended precision
    Rl = Rg.astype(np.longdouble)
    E = Rl.T @ Rl - (A.astype(np.longdouble) + s * np.eye(30, dtype=np.longdouble))
    assert np.all(np.abs(E) <= 1.5 * gamma(31) * (np.abs(Rg).T @ np.abs(Rg)))


# ------------------------------------------------------------------ TRSM
@gpu
@pytest.mark.parametrize("m,n", [(1, 1), (31, 5), (1000, 16), (4097, 64), (10007, 128), (3001, 160), (3000, 200),
                                 (2049, 256), (2001, 264), (3001, 300), (1500, 321), (1800, 512)])
def test_trsm_integer_exact(m, n):
    rng = np.random.default_rng(m)
    Q = rng.integers(-9, 10, size=(m, n)).astype(float)
    R = np.triu(rng.integers(-3, 4, size=(n, n))).astype(float)
    R[np.diag_indices(n)] = 2.0 ** rng.integers(0, 3, size=n)
    X = Q @ R
    # the substitution path (SUBST); the inverse-diagonal path: tests/test_gpu_trsm_diag.py
    assert np.array_equal(host(sq.scqr3_trsm(dev(X), dev(R), trsm_diag=sq.TRSM_DIAG_SUBST)), Q)


@gpu
@pytest.mark.parametrize("m,n", [(777, 24), (5003, 128), (1500, 256), (1100, 400)])
def test_trsm_rowwise_backward_error(m, n):
    X = synth.randsvd(m, n, 1e8, seed=3)
    R = oracle.cholesky(oracle.gram(X), oracle.shift(m, n, 1.0))
    # componentwise T3 holds for substitution; the inverse-diagonal path is held to
    # the paper's normwise bound (reading D24) in tests/test_gpu_trsm_diag.py
    Qg = host(sq.scqr3_trsm(dev(X), dev(R), trsm_diag=sq.TRSM_DIAG_SUBST))
    Rl = R.astype(np.longdouble)
    res = np.abs(Qg.astype(np.longdouble) @ Rl - X.astype(np.longdouble))
    bound = 2 * gamma(n + 1) * (np.abs(Qg) @ np.abs(R))
    assert np.all(res <= bound)
    Qo = oracle.trsm_rows(X, R)
    assert np.max(np.abs(Qg - Qo)) <= 1e-6 * np.max(np.abs(Qo))   # kappa(R) ~ 1e5


# ------------------------------------------------------------------ end to end
def _compare(X, rg, ro, kappa, d=None, e=None):
    m, n = X.shape
    Qg, Rg = host(rg.Q), host(rg.R)
    assert rg.status == 0 and ro.status == 0
    assert np.max(np.abs(Rg - ro.R)) <= 1e-10 * np.max(np.abs(ro.R))
    if kappa <= 1e6:
        assert np.max(np.abs(Qg - ro.Q)) <= 1e-10 * np.max(np.abs(ro.Q))
    elif kappa <= 1e8:
        assert np.max(np.abs(Qg - ro.Q)) <= 10 * kappa * U * np.max(np.abs(ro.Q))
    assert np.array_equal(Rg, np.triu(Rg)) and np.all(np.diag(Rg) > 0)
    orth = oracle.orth_F(Qg, d, e)
    res = oracle.resid_F(X, Qg, Rg)
    assert orth <= 10 * n * U, orth
    assert res <= 10 * n * U, res
    return orth, res


@gpu
@pytest.mark.parametrize("m,n,kappa", [(2000, 16, 1e12), (300, 10, 1e15), (1000, 30, 1e12), (100, 100, 1e13),
                                       (5001, 64, 1e4), (20000, 128, 1e10), (8000, 100, 1e6), (4000, 150, 1e9), (4000, 256, 1e8),
                                       (3000, 512, 1e10),
                                       (3000, 1, 1.0), (17, 17, 1e3)])
def test_factor_parity(m, n, kappa):
    X = synth.randsvd(m, n, kappa, seed=0)
    rg = sq.scqr3_factor(dev(X))
    ro = oracle.scqr3(X)
    _compare(X, rg, ro, kappa)
    if kappa <= 1 / U / (96 * (m * n + n * (n + 1))):   # Alg. 3's proven regime
        assert [t["shifted"] for t in rg.trace] == [t.shifted for t in ro.trace]
    else:   # beyond it, breakdown decisions sit within rounding of a threshold: both valid
        assert rg.trace[0]["shifted"] and ro.trace[0].shifted


@gpu
def test_pr1_exact_trace_and_shift():
    """BASELINE config PR1: shifted, plain, plain; the same shift as the oracle up to rounding."""
    X = synth.randsvd(2000, 16, 1e12, seed=0)
    rg = sq.scqr3_factor(dev(X))
    ro = oracle.scqr3(X)
    assert rg.passes == ro.passes == 3
    assert rg.trace[0]["shift"] == pytest.approx(ro.trace[0].shift, rel=1e-12)
    # the input Grams of passes 1-2 are data-determined; pass 3's deviation from I is rounding
    # noise of Q_2 (different in every correct implementation), so only its regime is compared
    for tg, to in zip(rg.trace[:2], ro.trace[:2]):
        assert tg["dev_F"] == pytest.approx(to.dev_F, rel=1e-6)
    assert rg.trace[2]["dev_F"] <= 0.5 and ro.trace[2].dev_F <= 0.5
    _compare(X, rg, ro, 1e12)
    # unshifted CholeskyQR2 breaks down on the GPU too
    rp = sq.scqr3_factor(dev(X), shift_mode=sq.SHIFT_NONE, max_passes=2)
    assert rp.status == sq.EBREAKDOWN


@gpu
def test_fixed_shift_first_pass_matches_oracle():
    X = synth.randsvd(3000, 40, 1e11, seed=4)
    s = 1e-9
    rg = sq.scqr3_factor(dev(X), shift_mode=sq.SHIFT_FIXED, shift_value=s, max_passes=1)
    ro = oracle.scqr3(X, shift_mode=oracle.SHIFT_FIXED, shift_value=s, max_passes=1)
    assert rg.status == ro.status == sq.ENOCONV
    Rg = host(rg.R)
    assert np.max(np.abs(Rg - ro.R)) <= 1e-9 * np.max(np.abs(ro.R))


@gpu
@pytest.mark.parametrize("m,n", [(40003, 72), (10007, 40)])   # (n = 40: fused TRSM + Gram, bulk Q stores)
def test_inplace_and_ragged_and_determinism(m, n):
    X = synth.randsvd(m, n, 1e9, seed=8)
    Xd = dev(X)
    r1 = sq.scqr3_factor(Xd)
    Q1, R1 = host(r1.Q), host(r1.R)
    r2 = sq.scqr3_factor(Xd)
    assert np.array_equal(Q1, host(r2.Q)) and np.array_equal(R1, host(r2.R))
    Xi = dev(X)
    r3 = sq.scqr3_factor(Xi, inplace=True)
    assert r3.Q.data_ptr() == Xi.data_ptr()
    assert np.array_equal(host(r3.Q), Q1) and np.array_equal(host(r3.R), R1)


@gpu
def test_status_codes_and_errors():
    X = synth.randsvd(500, 8, 1e3, seed=0)
    assert sq.scqr3_factor(dev(X), max_passes=1).status == sq.ENOCONV
    Z = np.zeros((300, 4))
    assert sq.scqr3_factor(dev(Z)).status in (sq.EBREAKDOWN, sq.ENOCONV)
    with pytest.raises(sq.ScqrError):
        sq.scqr3_factor(dev(np.ones((3, 5))))          # m < n
    with pytest.raises(sq.ScqrError):
        sq.scqr3_factor(dev(np.ones((600, 513))))      # n > 512


@gpu
@pytest.mark.parametrize("m,n,kappa", [(3000, 16, 1e12), (20000, 64, 1e12), (5000, 128, 1e8)])
def test_factor_oblique_parity(m, n, kappa):
    X = synth.randsvd(m, n, kappa, seed=1)
    d, e = synth.tridiag_b(m, seed=1)
    rg = sq.scqr3_factor_oblique(dev(X), torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda())
    ro = oracle.scqr3(X, d, e)
    _compare(X, rg, ro, kappa, d, e)


@gpu
def test_host_api_matches_device_api():
    X = synth.randsvd(10001, 48, 1e10, seed=2)
    rd = sq.scqr3_factor(dev(X))
    Xh = torch.from_numpy(np.asfortranarray(X)).t().contiguous().t()
    rh = sq.scqr3_factor_host(Xh)
    assert rh.status == 0
    assert np.array_equal(rh.R.numpy(), host(rd.R))
    assert np.array_equal(np.asarray(rh.Q.numpy()), host(rd.Q))


@gpu
@pytest.mark.parametrize("count", [1, 2, 5])
def test_host_batch_matches_single_calls(count):
    """scqr3_factor_host_batch (uploads / downloads overlapped with the factorisations, three
    rotating staging buffers) gives every matrix the bits of its own scqr3_factor_host call; a
    matrix that breaks down reports its status without disturbing the others; a repeated input
    buffer gives repeated results."""
    m, n = 7001, 40
    Xs = [synth.randsvd(m, n, 10.0 ** (4 + 2 * i), seed=i) for i in range(count)]
    def pin(A=None, shape=(m, n)):   # pinned column-major host tensor
        T = torch.empty(shape[::-1], dtype=torch.float64, pin_memory=True)
        if A is not None:
            T.copy_(torch.from_numpy(np.ascontiguousarray(A.T)))
        return T.t()

    Xh = [pin(X) for X in Xs]
    Qh = [pin() for _ in range(count)]
    Rh = [pin(shape=(n, n)) for _ in range(count)]
    st = sq.scqr3_factor_host_batch(Xh, Qh, Rh)
    assert st == [0] * count
    for i in range(count):
        r1 = sq.scqr3_factor_host(Xh[i])
        assert np.array_equal(r1.R.numpy(), Rh[i].numpy()) and np.array_equal(r1.Q.numpy(), Qh[i].numpy())
    # a plain (unshifted) CholeskyQR breaks down at kappa = 1e12; the others are fine
    bad = pin(synth.randsvd(m, n, 1e12, seed=9))
    Xb = [Xh[0], bad, Xh[0]]
    Qb = [pin() for _ in range(3)]
    Rb = [pin(shape=(n, n)) for _ in range(3)]
    st = sq.scqr3_factor_host_batch(Xb, Qb, Rb, shift_mode=sq.SHIFT_NONE)
    assert st[1] == sq.EBREAKDOWN and st[0] == st[2] == 0, st
    assert np.array_equal(Rb[0].numpy(), Rb[2].numpy()) and np.array_equal(Qb[0].numpy(), Qb[2].numpy())


@gpu
def test_single_rank_nccl_comm_path():
    """One-rank NCCL communicator: exercises ncclAllReduce / send-recv plumbing on one GPU."""
    import ctypes
    from paper_1809_11085_b200 import _abi
    buf = ctypes.create_string_buffer(128)
    assert _abi.lib().scqr3_comm_unique_id(buf) == 0
    h = ctypes.c_void_p()
    assert _abi.lib().scqr3_comm_init(ctypes.byref(h), 1, buf.raw, 0) == 0
    comm = sq.Comm(h, 0, 1)
    X = synth.randsvd(6000, 32, 1e11, seed=3)
    a = sq.scqr3_factor(dev(X))
    b = sq.scqr3_factor(dev(X), comm=comm)
    assert np.array_equal(host(a.R), host(b.R))
    d, e = synth.tridiag_b(6000, seed=3)
    c1 = sq.scqr3_factor_oblique(dev(X), torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda())
    c2 = sq.scqr3_factor_oblique(dev(X), torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda(), comm=comm)
    assert np.array_equal(host(c1.R), host(c2.R))
    # deterministic mode (allgather + rank-ordered sum): same bits as the plain path at one rank
    b2 = sq.scqr3_factor(dev(X), comm=comm, deterministic=True)
    assert np.array_equal(host(a.R), host(b2.R)) and b2.passes == a.passes
    c3 = sq.scqr3_factor_oblique(dev(X), torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda(), comm=comm,
                                 deterministic=True)
    assert np.array_equal(host(c1.R), host(c3.R))
    # complex path with the communicator (Gram allreduce of the split matrix)
    Z = synth.randsvd_complex(3000, 12, 1e9, seed=4)
    z1 = sq.scqr3_factor_complex(zdev(Z))
    z2 = sq.scqr3_factor_complex(zdev(Z), comm=comm)
    assert z1.status == z2.status == 0 and np.array_equal(z1.R.cpu().numpy(), z2.R.cpu().numpy())
    comm.destroy()


@gpu
@pytest.mark.parametrize("mode", ["adaptive", "practical"])
@pytest.mark.parametrize("m,n,kappa", [(3000, 12, 1e5), (20000, 64, 1e5), (2000, 16, 1e12), (1000, 50, 1e15),
                                       (30000, 128, 1e10)])
def test_shift_policies_parity(mode, m, n, kappa):
    """ADAPTIVE (Alg. 2) and PRACTICAL (Remark P:1600-1606, reading D21) on the GPU
    against the oracle: same shift decisions where they are not within rounding of a
    threshold, R parity and the BJ accuracy target."""
    sm = {"adaptive": sq.SHIFT_ADAPTIVE, "practical": sq.SHIFT_PRACTICAL}[mode]
    X = synth.randsvd(m, n, kappa, seed=0)
    rg = sq.scqr3_factor(dev(X), shift_mode=sm)
    ro = oracle.scqr3(X, shift_mode=sm)
    _compare(X, rg, ro, kappa)
    if kappa <= 1e5:   # far below u^-1/2: CholeskyQR2 (adaptive) / tiny shift (practical)
        assert rg.passes == ro.passes == 2
        assert [t["shifted"] for t in rg.trace] == [t.shifted for t in ro.trace]
    if mode == "practical":   # pass 1 is always shifted (by s_p, or by the safe s after a
        assert rg.trace[0]["shifted"] and ro.trace[0].shifted   # breakdown within rounding)


# ------------------------------------------------------------------ sparse SPD metric (CSR)
def _csr_dev(B, halo=0):
    return sq.CsrMetric(torch.from_numpy(B[0]), torch.from_numpy(B[1]), torch.from_numpy(B[2]), halo=halo)


@gpu
@pytest.mark.parametrize("m,n,dens", [(3, 2, 6), (40, 5, 6), (513, 33, 6), (3000, 64, 6), (2900, 64, 2),
                                      (1025, 17, 1)])
def test_gram_oblique_csr_exact_integers(m, n, dens):
    """dens = 6 gives ~13 nonzeros per row (more than 12: the host picks the row-chunk kernel
    csr_y_kernel), dens <= 2 at most ~5 (the tile kernel, staged CSR arrays); m off the 256-row
    tile size leaves a ragged last tile."""
    rng = np.random.default_rng(3 * m + n)
    M = np.zeros((m, m), dtype=np.int64)
    k = min(m * dens, m * m)
    r, c = rng.integers(0, m, k), rng.integers(0, m, k)
    M[r, c] = rng.integers(-9, 10, k)
    M = np.triu(M, 1)
    M = M + M.T
    M[np.diag_indices(m)] = rng.integers(1, 40, m)
    rp, ci, cv = [0], [], []
    for i in range(m):
        cols = [i] + [int(j) for j in np.nonzero(M[i])[0] if j != i]
        ci += cols
        cv += [float(M[i, j]) for j in cols]
        rp.append(len(ci))
    B = (np.array(rp, dtype=np.int64), np.array(ci, dtype=np.int32), np.array(cv))
    Xi = rng.integers(-20, 21, size=(m, n))
    A, cs = sq.scqr3_gram_oblique_csr(dev(Xi.astype(float)), _csr_dev(B))
    assert np.array_equal(host(A), (Xi.T @ M @ Xi).astype(float))
    assert cs.item() == float((Xi ** 2).sum())


@gpu
def test_gram_oblique_csr_uneven_density_exact_integers():
    """A metric with a dense 200 x 200 block (~50 nonzeros per row) in an otherwise sparse matrix
    (~3 per row): 6 nonzeros per row overall, so the tile kernel runs; its first 256-row tile
    exceeds the shared-memory stage (CSR arrays from global memory), the others are staged."""
    m, n = 3000, 40
    rng = np.random.default_rng(77)
    M = np.zeros((m, m), dtype=np.int64)
    r, c = rng.integers(0, m, m), rng.integers(0, m, m)
    M[r, c] = rng.integers(-9, 10, m)
    blk = rng.integers(-9, 10, (200, 200)) * (rng.random((200, 200)) < 0.25)
    M[:200, :200] = blk
    M = np.triu(M, 1)
    M = M + M.T
    M[np.diag_indices(m)] = rng.integers(1, 40, m)
    rp, ci, cv = [0], [], []
    for i in range(m):
        cols = [i] + [int(j) for j in np.nonzero(M[i])[0] if j != i]
        ci += cols
        cv += [float(M[i, j]) for j in cols]
        rp.append(len(ci))
    assert rp[256] > 12 * 256 and rp[-1] <= 12 * m   # first tile unstaged, tile kernel chosen
    B = (np.array(rp, dtype=np.int64), np.array(ci, dtype=np.int32), np.array(cv))
    Xi = rng.integers(-20, 21, size=(m, n))
    A, cs = sq.scqr3_gram_oblique_csr(dev(Xi.astype(float)), _csr_dev(B))
    assert np.array_equal(host(A), (Xi.T @ M @ Xi).astype(float))
    assert cs.item() == float((Xi ** 2).sum())


@gpu
@pytest.mark.parametrize("nx,ny,n", [(60, 50, 12), (250, 200, 64), (100, 40, 128)])
def test_factor_oblique_csr_laplacian(nx, ny, n):
    """2-D Laplacian metric (stand-in for the paper's sparse SPD B): R parity with the oracle,
    B-orthogonality and residual at the BJ target."""
    m = nx * ny
    B = synth.laplacian2d(nx, ny, seed=3, wmax=1e2)
    X = synth.randsvd(m, n, 1e10, seed=1)
    rg = sq.scqr3_factor_oblique_csr(dev(X), _csr_dev(B))
    ro = oracle.scqr3(X, csr=B)
    assert rg.status == 0 and ro.status == 0
    Rg, Qg = host(rg.R), host(rg.Q)
    assert np.max(np.abs(Rg - ro.R)) <= 1e-10 * np.max(np.abs(ro.R))
    assert oracle.orth_F_csr(Qg, B) <= 10 * n * U
    assert oracle.resid_F(X, Qg, Rg) <= 10 * n * U
    assert rg.trace[0]["shifted"] and ro.trace[0].shifted


@gpu
def test_csr_tridiagonal_matches_banded_path():
    m, n = 20000, 32
    X = synth.randsvd(m, n, 1e12, seed=2)
    d, e = synth.tridiag_b(m, seed=2)
    a = sq.scqr3_factor_oblique(dev(X), torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda())
    b = sq.scqr3_factor_oblique_csr(dev(X), _csr_dev(synth.tridiag_csr(d, e)))
    assert a.status == b.status == 0 and a.passes == b.passes
    Ra, Rb = host(a.R), host(b.R)
    assert np.max(np.abs(Ra - Rb)) <= 1e-12 * np.max(np.abs(Ra))


@gpu
def test_csr_argument_errors():
    m, n = 100, 4
    X = dev(synth.random_rows(m, n, seed=1))
    rp, ci, cv = synth.laplacian2d(10, 10)
    bad = ci.copy()
    bad[5] = m + 3                       # outside [0, m) with halo 0
    with pytest.raises(sq.ScqrError):
        sq.scqr3_factor_oblique_csr(X, _csr_dev((rp, bad, cv)))
    with pytest.raises(sq.ScqrError):    # halo without a communicator
        sq.scqr3_factor_oblique_csr(X, _csr_dev((rp, ci, cv), halo=2))
    r = sq.scqr3_factor_oblique_csr(X, _csr_dev((rp, ci, cv)))
    assert r.status == 0


@gpu
@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_non_finite_input_raises(bad):
    X = synth.randsvd(3000, 16, 1e3, seed=1)
    X[1234, 7] = bad
    with pytest.raises(sq.ScqrError, match="non-finite"):
        sq.scqr3_factor(dev(X))
    r = sq.scqr3_factor(dev(synth.randsvd(3000, 16, 1e3, seed=1)))   # the context recovers
    assert r.status == 0


# ------------------------------------------------------------------ complex X (N4)
def zdev(Z):
    t = torch.from_numpy(np.asarray(Z, dtype=np.complex128))
    out = sq.colmajor_empty_complex(t.shape[0], t.shape[1])
    out.copy_(t)
    return out


@gpu
@pytest.mark.parametrize("m,n,kappa", [(2000, 16, 1e12), (300, 5, 1e3), (20000, 64, 1e10), (5000, 100, 1e8),
                                       (3000, 128, 1e12), (1500, 256, 1e6)])
def test_complex_factor_parity(m, n, kappa):
    X = synth.randsvd_complex(m, n, kappa, seed=0)
    rg = sq.scqr3_factor_complex(zdev(X))
    ro = oracle.zscqr3(X)
    assert rg.status == 0 and ro.status == 0
    Rg, Qg = rg.R.cpu().numpy(), rg.Q.cpu().numpy()
    assert np.max(np.abs(Rg - ro.R)) <= 1e-10 * np.max(np.abs(ro.R))
    assert np.array_equal(Rg, np.triu(Rg)) and np.all(np.diag(Rg).real > 0) and not np.diag(Rg).imag.any()
    assert oracle.zorth_F(Qg) <= 10 * n * U
    assert oracle.zresid_F(X, Qg, Rg) <= 10 * n * U
    assert rg.trace[0]["shifted"] and ro.trace[0].shifted


@gpu
def test_complex_real_input_matches_real_path():
    X = synth.randsvd(4000, 24, 1e10, seed=3)
    a = sq.scqr3_factor(dev(X))
    b = sq.scqr3_factor_complex(zdev(X.astype(np.complex128)))
    assert a.status == b.status == 0 and a.passes == b.passes
    Ra, Rb = host(a.R), b.R.cpu().numpy()
    assert np.max(np.abs(Rb.imag)) == 0.0
    assert np.max(np.abs(Ra - Rb.real)) <= 1e-12 * np.max(np.abs(Ra))


# Complex n in (256, 512]: the 2n-column split matrix as [S1 S2] (zwide.cu) -- the real Gram and
# TRSM on each block, the cross Gram S1^T S2 and the block update S2 -= Q1 M12 (P:124-125,
# P:323-334 row-wise; reading D23).  Ragged m (not a multiple of 32 or 64), several cross-Gram
# chunks and update row blocks, q = 2n - 512 off the 64-column blocks.
@gpu
@pytest.mark.parametrize("m,n,kappa", [(3001, 260, 1e8), (9999, 300, 1e12), (4003, 384, 1e10), (2500, 512, 1e6)])
def test_complex_wide_factor_parity(m, n, kappa):
    X = synth.randsvd_complex(m, n, kappa, seed=1)
    rg = sq.scqr3_factor_complex(zdev(X))
    ro = oracle.zscqr3(X)
    assert rg.status == 0 and ro.status == 0
    Rg, Qg = rg.R.cpu().numpy(), rg.Q.cpu().numpy()
    assert np.max(np.abs(Rg - ro.R)) <= 1e-10 * np.max(np.abs(ro.R))
    assert np.array_equal(Rg, np.triu(Rg)) and np.all(np.diag(Rg).real > 0) and not np.diag(Rg).imag.any()
    assert oracle.zorth_F(Qg) <= 10 * n * U
    assert oracle.zresid_F(X, Qg, Rg) <= 10 * n * U
    assert rg.trace[0]["shifted"] and ro.trace[0].shifted


@gpu
@pytest.mark.parametrize("n", [300, 512])
def test_complex_wide_real_input_matches_real_path(n):
    """A real X through the wide complex path: imaginary parts exactly zero, R equal to the real
    path's (an independent route: the real kernels on the n columns of X itself)."""
    X = synth.randsvd(6000, n, 1e9, seed=5)
    a = sq.scqr3_factor(dev(X))
    b = sq.scqr3_factor_complex(zdev(X.astype(np.complex128)))
    assert a.status == b.status == 0
    Ra, Rb = host(a.R), b.R.cpu().numpy()
    assert np.max(np.abs(Rb.imag)) == 0.0
    assert np.max(np.abs(Ra - Rb.real)) <= 1e-12 * np.max(np.abs(Ra))
    assert np.max(np.abs(b.Q.cpu().numpy().imag)) == 0.0


@gpu
def test_complex_wide_deterministic_and_inplace_blocks():
    """Two calls give the same bits (fixed-order cross-Gram reduction); the SUBST and INVERSE
    diagonal modes both reach the oracle's R."""
    X = synth.randsvd_complex(5000, 280, 1e10, seed=2)
    a = sq.scqr3_factor_complex(zdev(X))
    b = sq.scqr3_factor_complex(zdev(X))
    c = sq.scqr3_factor_complex(zdev(X), trsm_diag=sq.TRSM_DIAG_SUBST)
    assert a.status == b.status == c.status == 0
    assert np.array_equal(a.R.cpu().numpy(), b.R.cpu().numpy())
    assert np.array_equal(a.Q.cpu().numpy(), b.Q.cpu().numpy())
    ro = oracle.zscqr3(X)
    for r in (a, c):
        assert np.max(np.abs(r.R.cpu().numpy() - ro.R)) <= 1e-10 * np.max(np.abs(ro.R))


@gpu
@pytest.mark.parametrize("m,n,col", [(3000, 200, 137), (4000, 300, 290), (2000, 160, 3)])
def test_complex_blocked_cholesky_breakdown_pivot(m, n, col):
    """The blocked complex Cholesky (W in global memory, n > 128): a zero column makes the
    unshifted Gram's pivot exactly 0 at that column (S:69 breakdown = pivot <= 0), on the GPU and
    in the oracle; with the shift the factorisation goes through (pivot index is 1-based)."""
    X = synth.randsvd_complex(m, n, 1e4, seed=3)
    X[:, col] = 0
    rg = sq.scqr3_factor_complex(zdev(X), shift_mode=sq.SHIFT_NONE, max_passes=2)
    ro = oracle.zscqr3(X, shift_mode=oracle.SHIFT_NONE, max_passes=2)
    assert rg.status == sq.EBREAKDOWN and ro.status == sq.EBREAKDOWN
    assert rg.trace[0]["breakdown_pivot"] == ro.trace[0].breakdown_pivot == col + 1
    assert rg.trace[0]["pivot_value"] == 0.0


# ------------------------------------------------------------------ wide TRSM, several sweeps
# One persistent sweep of the TRSM covers 148 CTAs x 8 warps x 16 rows = 18,944 rows; at
# m >= 60,000 every block-column launch of the n in (128, 512] path (columns 0..127, targets
# 16..17 / 16..19 / 16..21 / 16..23 / 16..27 / 16..31, and for n > 256 the resident launches 32..40 ... 60..64) runs at least three
# sweeps per warp, so their loop-carried state (TMA slot reuse, resident fragments, the read-back
# of finished Q columns) is compared with the oracle (the per-row model).
@gpu
@pytest.mark.parametrize("n", [136, 144, 150, 176, 192, 200, 300, 400, 512])
def test_trsm_integer_exact_full_sweeps(n):
    m = 60_011
    rng = np.random.default_rng(n + 1)
    Q = rng.integers(-9, 10, size=(m, n)).astype(float)
    R = np.triu(rng.integers(-3, 4, size=(n, n))).astype(float)
    R[np.diag_indices(n)] = 2.0 ** rng.integers(0, 3, size=n)
    X = Q @ R
    assert np.array_equal(host(sq.scqr3_trsm(dev(X), dev(R), trsm_diag=sq.TRSM_DIAG_SUBST)), Q)


@gpu
@pytest.mark.parametrize("n,kappa", [(136, 1e10), (150, 1e9), (192, 1e10), (200, 1e12), (300, 1e8), (400, 1e10),
                                     (512, 1e12)])
def test_factor_parity_full_sweeps(n, kappa):
    m = 60_000
    X = synth.randsvd(m, n, kappa, seed=7)
    rg = sq.scqr3_factor(dev(X))
    ro = oracle.scqr3(X)
    _compare(X, rg, ro, kappa)


# ------------------------------------------------------------------ round-2 paths
@gpu
@pytest.mark.parametrize("m,n", [(60_001, 150), (40_000, 192), (33_333, 176)])
def test_gram_parity_cluster_multicast(m, n):
    """n in (128, 192]: two CTAs share each row chunk and run as a thread-block cluster whose
    stages arrive by TMA multicast (gram.cu); T1 bound against the oracle, exact symmetry."""
    X = synth.random_rows(m, n, seed=n)
    A = host(sq.scqr3_gram(dev(X)))
    Ao = oracle.gram(X)
    bound = 2 * gamma(m) * (np.abs(X).T @ np.abs(X))
    assert np.all(np.abs(A - Ao) <= bound + 1e-300)
    assert np.array_equal(A, A.T)
    Xi = np.random.default_rng(n).integers(-30, 31, size=(m, n)).astype(float)
    Ai = host(sq.scqr3_gram(dev(Xi)))
    assert np.array_equal(Ai, (Xi.astype(np.int64).T @ Xi.astype(np.int64)).astype(float))


@gpu
@pytest.mark.parametrize("n", [136, 200, 256])
def test_cluster_power_iteration_shift(n):
    """n in (128, 256]: pass 1's norm estimate comes from power_cluster_kernel (8 CTAs); the
    shift equals the oracle's (the same 32-step power iteration, reading D2) to rounding."""
    m = 20_000
    X = synth.randsvd(m, n, 1e10, seed=n)
    rg = sq.scqr3_factor(dev(X))
    ro = oracle.scqr3(X)
    assert rg.status == 0 and ro.status == 0
    assert rg.trace[0]["norm2_est"] == pytest.approx(ro.trace[0].norm2_est, rel=1e-12)
    assert rg.trace[0]["shift"] == pytest.approx(ro.trace[0].shift, rel=1e-12)
    _compare(X, rg, ro, 1e10)
