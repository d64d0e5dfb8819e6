"""Pins for the oracle's building blocks (CPU only).  Every test checks the oracle against
something other than itself: exact integer arithmetic, exact rationals, closed forms, the
paper's error bounds evaluated exactly, or an independent library routine."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

U = 2.0 ** -53
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def gamma(k):
    return k * U / (1 - k * U)


def exact_mat(A):
    return [[Fraction(float(x)) for x in row] for row in np.asarray(A)]


def exact_matmul(A, B):
    n, k, p = len(A), len(B), len(B[0])
    return [[sum((A[i][l] * B[l][j] for l in range(k)), Fraction(0)) for j in range(p)] for i in range(n)]


# --------------------------------------------------------------------------- Gram
def test_gram_spec_examples():
    assert np.array_equal(oracle.gram(np.eye(3)), np.eye(3))
    g = GOLD["gram_ones"]
    assert np.array_equal(oracle.gram(np.array(g["X"], float)), np.array(g["A"], float))


@pytest.mark.parametrize("m,n", [(1, 1), (7, 3), (200, 17), (1000, 33)])
def test_gram_exact_integers(m, n):
    rng = np.random.default_rng(m * 100 + n)
    Xi = rng.integers(-50, 51, size=(m, n))
    A = oracle.gram(Xi.astype(float))
    ref = Xi.T.astype(np.int64) @ Xi.astype(np.int64)   # exact; |entries| << 2^53
    assert np.array_equal(A, ref.astype(float))
    assert np.array_equal(A, A.T)


def test_gram_componentwise_T1_bound():
    """|fl(X^T X) - X^T X| <= gamma_m |X|^T |X|, exact rationals."""
    X = synth.randsvd(60, 5, 1e6, seed=3)
    A = oracle.gram(X)
    Xe = exact_mat(X)
    XeT = [list(r) for r in zip(*Xe)]
    exact = exact_matmul(XeT, Xe)
    absX = np.abs(X)
    bound = gamma(60) * (absX.T @ absX)
    for j in range(5):
        for l in range(5):
            err = abs(Fraction(float(A[j, l])) - exact[j][l])
            assert err <= Fraction(float(bound[j, l])) * Fraction(1001, 1000)
    assert np.array_equal(A, A.T)


def test_gram_oblique_identity_metric_equals_gram():
    """B = I: every oblique step degenerates -- bitwise here."""
    X = synth.random_rows(300, 9, seed=1)
    A, cs = oracle.gram_oblique(X, np.ones(300), np.zeros(300))
    assert np.array_equal(A, oracle.gram(X))
    assert np.allclose(cs, np.diag(oracle.gram(X)), rtol=0, atol=0)


@pytest.mark.parametrize("m,n", [(2, 1), (9, 4), (150, 7)])
def test_gram_oblique_exact_integers(m, n):
    rng = np.random.default_rng(m + 17 * n)
    Xi = rng.integers(-20, 21, size=(m, n))
    d = rng.integers(1, 40, size=m)
    e = rng.integers(-9, 10, size=m)
    e[-1] = 0
    B = np.diag(d) + np.diag(e[:-1], 1) + np.diag(e[:-1], -1)
    ref = Xi.T.astype(np.int64) @ B.astype(np.int64) @ Xi.astype(np.int64)
    A, cs = oracle.gram_oblique(Xi.astype(float), d.astype(float), e.astype(float))
    assert np.array_equal(A, ref.astype(float))
    assert np.array_equal(cs, (Xi.astype(np.int64) ** 2).sum(0).astype(float))


def _random_sym_csr(m, rng, density=0.05):
    """Random symmetric integer sparse matrix as CSR (diagonal first, then ascending)."""
    M = np.zeros((m, m), dtype=np.int64)
    mask = np.triu(rng.random((m, m)) < density, 1)
    M[mask] = rng.integers(-9, 10, size=mask.sum())
    M = M + M.T
    M[np.diag_indices(m)] = rng.integers(1, 40, size=m)
    rp, ci, cv = [0], [], []
    for i in range(m):
        cols = [i] + [j for j in range(m) if j != i and M[i, j] != 0]
        ci += cols
        cv += [float(M[i, j]) for j in cols]
        rp.append(len(ci))
    return M, (np.array(rp), np.array(ci), np.array(cv))


@pytest.mark.parametrize("m,n", [(3, 2), (40, 5), (120, 9)])
def test_gram_oblique_csr_exact_integers(m, n):
    """General sparse B: integer X and B keep every product and sum exact,
    so the result must equal int64 arithmetic X^T B X bit for bit."""
    rng = np.random.default_rng(3 * m + n)
    M, B = _random_sym_csr(m, rng)
    Xi = rng.integers(-20, 21, size=(m, n))
    ref = Xi.T @ M @ Xi
    A, cs = oracle.gram_oblique_csr(Xi.astype(float), B)
    assert np.array_equal(A, ref.astype(float))
    assert np.array_equal(cs, (Xi ** 2).sum(0).astype(float))


def test_gram_oblique_csr_tridiagonal_and_identity():
    """The tridiagonal metric written as CSR in the banded term order is the same operation
    (bitwise equal to the pinned banded Gram); the CSR identity gives the plain Gram."""
    X = synth.random_rows(700, 11, seed=4)
    d, e = synth.tridiag_b(700, seed=2)
    A1, c1 = oracle.gram_oblique(X, d, e)
    A2, c2 = oracle.gram_oblique_csr(X, synth.tridiag_csr(d, e))
    assert np.array_equal(A1, A2) and np.array_equal(c1, c2)
    eye = (np.arange(701), np.arange(700, dtype=np.int32), np.ones(700))
    A3, _ = oracle.gram_oblique_csr(X, eye)
    assert np.array_equal(A3, oracle.gram(X))
    Q = synth.random_rows(700, 6, seed=5)
    # (the metric's final sum over entries is an OpenMP reduction: equal up to its order)
    a, b = oracle.orth_F_csr(Q, synth.tridiag_csr(d, e)), oracle.orth_F(Q, d, e)
    assert abs(a - b) <= 1e-14 * b


# --------------------------------------------------------------------------- Cholesky
def test_cholesky_spec_examples():
    g = GOLD["chol_25_20"]
    assert np.array_equal(oracle.cholesky(np.array(g["A"], float)), np.array(g["R"], float))
    g = GOLD["chol_singular"]
    r = oracle.cholesky(np.array(g["A"], float))
    assert isinstance(r, oracle.Breakdown) and r.pivot == g["pivot"] and r.value <= 0
    assert np.array_equal(oracle.cholesky(np.eye(4)), np.eye(4))


@pytest.mark.parametrize("n", [1, 2, 5, 12, 40])
def test_cholesky_recovers_integer_factor_exactly(n):
    """A = R^T R with integer R (positive diagonal): every pivot is a perfect square and every
    division exact, so an index/transpose slip cannot survive."""
    rng = np.random.default_rng(n)
    R = np.triu(rng.integers(-6, 7, size=(n, n))).astype(float)
    R[np.diag_indices(n)] = rng.integers(1, 9, size=n)
    A = R.T @ R
    assert np.array_equal(oracle.cholesky(A), R)


def test_cholesky_shift_is_added_to_the_diagonal():
    R = np.array([[2.0, 1.0, -3.0], [0, 3.0, 2.0], [0, 0, 1.0]])
    A = R.T @ R
    assert np.array_equal(oracle.cholesky(A - 5.0 * np.eye(3), 5.0), R)


def test_cholesky_breakdown_index_and_value():
    A = np.diag([1.0, 2.0, -1.0, 3.0])
    r = oracle.cholesky(A)
    assert isinstance(r, oracle.Breakdown) and r.pivot == 3 and r.value == -1.0
    A = np.diag([1.0, np.nan, 1.0])
    r = oracle.cholesky(A)
    assert isinstance(r, oracle.Breakdown) and r.pivot == 2
    # the first breakdown of CholeskyQR on an ill-conditioned Gram
    X = synth.randsvd(1000, 30, 1e12, seed=1)
    assert isinstance(oracle.cholesky(oracle.gram(X)), oracle.Breakdown)


def test_cholesky_T2_backward_error_exact():
    """|R^T R - (A + sI)| <= gamma_{n+1} |R^T||R|, exact rationals."""
    X = synth.randsvd(40, 8, 1e3, seed=5)
    A = oracle.gram(X)
    s = 1e-3
    R = oracle.cholesky(A, s)
    Re = exact_mat(R)
    RtR = exact_matmul([list(r) for r in zip(*Re)], Re)
    bound = gamma(9) * (np.abs(R).T @ np.abs(R))
    for i in range(8):
        for j in range(8):
            target = Fraction(float(A[i, j])) + (Fraction(s) if i == j else 0)
            assert abs(RtR[i][j] - target) <= Fraction(float(bound[i, j])) * Fraction(1001, 1000)
    assert np.all(np.diag(R) > 0) and np.array_equal(R, np.triu(R))


def test_cholesky_T4_weyl_shift_bound():
    """sigma_n(R)^2 >= sigma_n(X)^2 + 0.9 s."""
    X = synth.randsvd(300, 12, 1e14, seed=2)
    s = oracle.shift(300, 12, 1.0)
    R = oracle.cholesky(oracle.gram(X), s)
    sx = np.linalg.svd(X, compute_uv=False)[-1]
    sr = np.linalg.svd(R, compute_uv=False)[-1]
    assert sr ** 2 >= sx ** 2 + 0.9 * s


# --------------------------------------------------------------------------- TRSM
def test_trsm_spec_example():
    g = GOLD["trsm_hand"]
    Q = oracle.trsm_rows(np.array(g["X"], float), np.array(g["R"], float))
    assert np.array_equal(Q, np.array(g["Q"], float))


@pytest.mark.parametrize("m,n", [(1, 1), (33, 6), (500, 24)])
def test_trsm_exact_integer(m, n):
    """X = Q R with integer Q and integer R whose diagonal is +-powers of two: every
    substitution step is exact, so Q must come back bit for bit."""
    rng = np.random.default_rng(m + n)
    Q = rng.integers(-9, 10, size=(m, n)).astype(float)
    R = np.triu(rng.integers(-4, 5, size=(n, n))).astype(float)
    R[np.diag_indices(n)] = 2.0 ** rng.integers(0, 3, size=n)
    X = Q @ R
    assert np.array_equal(oracle.trsm_rows(X, R), Q)


def test_trsm_T3_rowwise_backward_error_exact():
    """|q_i R - x_i| <= gamma_n |q_i| |R| row by row."""
    X = synth.randsvd(30, 7, 1e5, seed=4)
    R = oracle.cholesky(oracle.gram(X), 1e-8)
    Q = oracle.trsm_rows(X, R)
    Re = exact_mat(R)
    absR = np.abs(R)
    for i in range(30):
        qi = [Fraction(float(v)) for v in Q[i]]
        bnd = gamma(7) * (np.abs(Q[i]) @ absR)
        for j in range(7):
            r = sum((qi[l] * Re[l][j] for l in range(7)), Fraction(0)) - Fraction(float(X[i, j]))
            assert abs(r) <= Fraction(float(bnd[j])) * Fraction(1001, 1000)


# --------------------------------------------------------------------------- trmul
def test_trmul():
    g = GOLD["trmul_diag"]
    assert np.array_equal(oracle.trmul(np.array(g["R1"], float), np.array(g["R2"], float)),
                          np.array(g["P"], float))
    rng = np.random.default_rng(0)
    A = np.triu(rng.integers(-9, 10, size=(11, 11))).astype(float)
    B = np.triu(rng.integers(-9, 10, size=(11, 11))).astype(float)
    assert np.array_equal(oracle.trmul(A, B), A @ B)


# --------------------------------------------------------------------------- norm estimate / shift
def test_power_lmax_closed_forms():
    # diag(3,1,2) from the all-ones start: after k steps x ~ (3^k, 1, 2^k), so the Rayleigh
    # quotient is (3^(2k+1) + 1 + 2^(2k+1)) / (3^(2k) + 1 + 2^(2k)) exactly.
    for k in (1, 5, 32):
        rq = Fraction(3 ** (2 * k + 1) + 1 + 2 ** (2 * k + 1), 3 ** (2 * k) + 1 + 2 ** (2 * k))
        assert oracle.power_lmax(np.diag([3.0, 1.0, 2.0]), iters=k) == pytest.approx(float(rq), rel=1e-14)
    u = np.array([1.0, -2.0, 0.5, 4.0])
    lam = oracle.power_lmax(np.outer(u, u), iters=1)   # exact after one step on a rank-one Gram
    assert lam == pytest.approx(u @ u, rel=1e-14)
    X = synth.randsvd(200, 10, 1e4, seed=9)
    A = oracle.gram(X)
    assert oracle.power_lmax(A) == pytest.approx(np.linalg.eigvalsh(A)[-1], rel=1e-12)


def test_shift_values_and_homogeneity():
    for key in ("shift_1000_30", "shift_1_1"):
        g = GOLD[key]
        assert oracle.shift(g["m"], g["n"], 1.0) == pytest.approx(g["s"], rel=1e-3)
    g = GOLD["shift_oblique_300_30"]
    assert oracle.shift_oblique(g["m"], g["n"], 1.0, 1.0) == pytest.approx(g["s"], rel=1e-3)
    assert oracle.shift(1000, 30, 4.0) == 4 * oracle.shift(1000, 30, 1.0)
    assert oracle.shift_oblique(300, 30, 1.0, 2.0) == 2 * oracle.shift_oblique(300, 30, 1.0, 1.0)
    # exact formula 11(mn + n(n+1)) 2^-53
    assert oracle.shift(1000, 30, 1.0) == 11 * (1000 * 30 + 30 * 31) * 2.0 ** -53
    # oblique dominates the standard shift (2m sqrt(mn) >= mn)
    for m, n in [(10, 10), (1000, 3), (5, 1)]:
        assert oracle.shift_oblique(m, n, 1, 1) >= oracle.shift(m, n, 1)


# --------------------------------------------------------------------------- metrics (F6, D13)
def test_metrics_exact_cases():
    Q = np.eye(5)[:, :3]
    assert oracle.orth_F(Q) == 0.0
    Q2 = Q.copy()
    Q2[0, 0] = 2.0      # Q^T Q - I has a single entry 3
    assert oracle.orth_F(Q2) == 3.0
    X = np.array([[3.0, 0.0], [4.0, 5.0]])
    Qx = np.array([[0.6, -0.8], [0.8, 0.6]])
    R = np.array([[5.0, 4.0], [0.0, 3.0]])
    assert oracle.resid_F(X, Qx, R) < 4 * U
    d = np.array([4.0, 9.0, 1.0])
    e = np.zeros(3)
    Qb = np.diag(1 / np.sqrt(d))[:, :2]
    assert oracle.orth_F(Qb, d, e) < 4 * U
