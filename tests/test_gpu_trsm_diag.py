"""The TRSM's inverse-diagonal path and its guard (reading D24).

The paper's analysis needs, for every row, (R~ + dR_i) q_i = x_i with ||dR_i||_2 <=
gamma_n sqrt(n) ||R~||_2 (eq. DeltaRbound).  Substitution gives the stronger
componentwise |dR_i| <= gamma_n |R~| (tests/test_gpu_parity.py).  The inverse path
multiplies each row's 8-column block by Y_J = D_J^{-1}; the Cholesky step enables it only when
    gamma_n ||R~_off||_F + 2 gamma_8 max_J || |D_J||Y_J||D_J| ||_F <= gamma_n sqrt(n) max_j ||R~ e_j||_2 .
Pinned here:
  * exactness of the inverse path's data layout on integer cases whose Y_J are dyadic
    (D_J = diag(2^k)(I + N), N strictly upper integer: Y_J = (I + N)^{-1} diag(2^-k) exactly);
  * the guard's decision: AUTO reproduces the forced-INVERSE bits when the criterion (evaluated
    here in numpy, far from the threshold) holds and the SUBST bits when it fails;
  * the normwise per-row bound on the AUTO result in extended precision;
  * factorisations through the inverse path against the oracle (R, orthogonality, residual).
"""
import numpy as np
import pytest
import scipy.linalg as sl

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


def guard_ratio(R):
    """lhs / rhs of the D24 criterion (the device evaluates the same quantities)."""
    n = R.shape[0]
    mus, off = [], R.copy()
    for J in range(0, n, 8):
        D = R[J:J + 8, J:J + 8]
        Y = sl.solve_triangular(D.T, np.eye(D.shape[0]), lower=True).T
        mus.append(np.linalg.norm(np.abs(D) @ np.abs(Y) @ np.abs(D)))
        off[J:J + 8, J:J + 8] = 0
    lhs = gamma(n) * np.linalg.norm(off) + 2 * gamma(8) * max(mus)
    rhs = gamma(n) * np.sqrt(n) * np.linalg.norm(R, axis=0).max()
    return lhs / rhs


def dyadic_blocks(n, rng):
    R = np.triu(rng.integers(-3, 4, size=(n, n))).astype(float)
    for J in range(0, n, 8):
        b = min(8, n - J)
        N = np.triu(rng.integers(-1, 2, size=(b, b)), 1).astype(float)
        R[J:J + b, J:J + b] = np.diag(2.0 ** rng.integers(0, 3, size=b)) @ (np.eye(b) + N)
    return R


@gpu
@pytest.mark.parametrize("m,n", [(1, 96), (999, 72), (3001, 96), (60_011, 128), (10_007, 136), (60_011, 256),
                                 (3001, 300)])
def test_trsm_inverse_integer_exact(m, n):
    """Forced INVERSE: every row solved through Y_J fragments (several persistent sweeps at m=60011).
    (The kernel-level TRSM has inverse instances for n > 64; n in (32, 64] has one only fused with
    the next pass's Gram inside scqr3_factor, covered by test_factor_inverse_path_parity.)"""
    rng = np.random.default_rng(m + n)
    Q = rng.integers(-9, 10, size=(m, n)).astype(float)
    R = dyadic_blocks(n, rng)
    X = Q @ R
    assert np.array_equal(host(sq.scqr3_trsm(dev(X), dev(R), trsm_diag=sq.TRSM_DIAG_INVERSE)), Q)


def _shifted_R(m, n, kappa, seed):
    X = synth.randsvd(m, n, kappa, seed=seed)
    return X, oracle.cholesky(oracle.gram(X), oracle.shift(m, n, 1.0))


@gpu
@pytest.mark.parametrize("m,n,kappa", [(5003, 72, 1e12), (5003, 96, 1e8), (20_000, 128, 1e10), (3000, 200, 1e10)])
def test_guard_takes_inverse_when_bound_holds(m, n, kappa):
    X, R = _shifted_R(m, n, kappa, 5)
    assert guard_ratio(R) < 0.8
    Xd, Rd = dev(X), dev(R)
    qa = host(sq.scqr3_trsm(Xd, Rd))
    qi = host(sq.scqr3_trsm(Xd, Rd, trsm_diag=sq.TRSM_DIAG_INVERSE))
    qs = host(sq.scqr3_trsm(Xd, Rd, trsm_diag=sq.TRSM_DIAG_SUBST))
    assert np.array_equal(qa, qi)
    assert not np.array_equal(qa, qs)   # the two paths round differently
    # eq. (DeltaRbound): ||x_i - q_i R||_2 <= gamma_n sqrt(n) ||R||_2 ||q_i||_2, per row
    res = np.sqrt((((qa.astype(np.longdouble) @ R.astype(np.longdouble)) - X.astype(np.longdouble)) ** 2).sum(1))
    bound = gamma(n) * np.sqrt(n) * np.linalg.norm(R, 2) * np.linalg.norm(qa, axis=1)
    assert np.all(res.astype(float) <= bound)
    Qo = oracle.trsm_rows(X, R)
    assert np.max(np.abs(qa - Qo)) <= 1e-6 * np.max(np.abs(Qo))


@gpu
@pytest.mark.parametrize("n", [96, 128, 256])
def test_guard_falls_back_to_substitution(n):
    """One ill-conditioned diagonal block (mu_J ~ 1e8 ||D_J||): AUTO must be the substitution bits."""
    m = 4001
    X, R = _shifted_R(m, n, 1e6, 7)
    J = 8 * (n // 16)
    R[J, J + 1] = 1e4 * R[J + 1, J + 1]
    R[J + 1, J + 2] = 1e4 * R[J + 2, J + 2]
    assert guard_ratio(R) > 10
    Xd, Rd = dev(X), dev(R)
    qa = host(sq.scqr3_trsm(Xd, Rd))
    qs = host(sq.scqr3_trsm(Xd, Rd, trsm_diag=sq.TRSM_DIAG_SUBST))
    assert np.array_equal(qa, qs)


@gpu
@pytest.mark.parametrize("n", [16, 64])
def test_guard_small_n_substitutes(n):
    """n = 16 (PR1's width: gamma_n sqrt(n) leaves no room, ratio ~3.5 on pass 1) and the kernel-level
    n <= 64 have no inverse instance -- AUTO, INVERSE and SUBST give the same bits."""
    X, R = _shifted_R(2000, n, 1e12, 0)
    Xd, Rd = dev(X), dev(R)
    qs = host(sq.scqr3_trsm(Xd, Rd, trsm_diag=sq.TRSM_DIAG_SUBST))
    assert np.array_equal(host(sq.scqr3_trsm(Xd, Rd)), qs)
    assert np.array_equal(host(sq.scqr3_trsm(Xd, Rd, trsm_diag=sq.TRSM_DIAG_INVERSE)), qs)


@gpu
@pytest.mark.parametrize("m,n,kappa", [(60_000, 64, 1e15), (60_000, 128, 1e10), (30_000, 96, 1e12), (30_000, 256, 1e14)])
def test_factor_inverse_path_parity(m, n, kappa):
    """Factorisations whose guard passes on every pass (AUTO == forced INVERSE bit for bit), against
    the oracle: R within 1e-10 max|R|, orthogonality and residual <= 10 n u (reading D14)."""
    X = synth.randsvd(m, n, kappa, seed=1, spectrum="cluster" if n == 256 else "geometric")
    Xd = dev(X)
    ra = sq.scqr3_factor(Xd)
    ri = sq.scqr3_factor(Xd, trsm_diag=sq.TRSM_DIAG_INVERSE)
    rs = sq.scqr3_factor(Xd, trsm_diag=sq.TRSM_DIAG_SUBST)
    assert ra.status == ri.status == rs.status == 0
    assert np.array_equal(host(ra.R), host(ri.R)) and np.array_equal(host(ra.Q), host(ri.Q))
    assert not np.array_equal(host(ra.Q), host(rs.Q))   # AUTO did take the inverse path
    ro = oracle.scqr3(X)
    for r in (ra, rs):
        Rg, Qg = host(r.R), host(r.Q)
        assert np.max(np.abs(Rg - ro.R)) <= 1e-10 * np.max(np.abs(ro.R))
        assert oracle.orth_F(Qg) <= 10 * n * U
        assert oracle.resid_F(X, Qg, Rg) <= 10 * n * U
