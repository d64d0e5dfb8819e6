"""End-to-end pins for the oracle's pass controller (Alg. 3 + Alg. 2 re-shift, readings D2-D8).

Independent references: exact tiny QR, LAPACK Householder QR (numpy), the paper's theorem
ceilings, the exact-arithmetic closed form of the first pass
(P:555-563), the paper's Tables 1-3 (orders of magnitude, tests/golden/paper_tables.json),
and the breakdown of unshifted CholeskyQR2 that motivates the method."""
import json
import os

import numpy as np
import pytest

import oracle
import synth

U = 2.0 ** -53
TABLES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables.json")))
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def householder_R(X):
    """LAPACK Householder QR, sign-normalised so diag(R) > 0."""
    Q, R = np.linalg.qr(X)
    s = np.sign(np.diag(R))
    return Q * s, R * s[:, None]


def test_exact_tiny_qr():
    g = GOLD["qr_3_4"]
    r = oracle.scqr3(np.array(g["X"], float))
    assert r.status == 0
    assert np.allclose(r.R, np.array(g["R"]), rtol=0, atol=20 * U * 5)
    assert np.allclose(r.Q, np.array(g["Q"]), rtol=0, atol=20 * U)


def test_orthogonal_columns_give_diagonal_R():
    rng = np.random.default_rng(3)
    Q0, _ = np.linalg.qr(rng.standard_normal((200, 6)))
    scales = np.array([3.0, 1.0, 0.5, 7.0, 2.0, 1e-3])
    r = oracle.scqr3(Q0 * scales)
    assert r.status == 0
    assert np.allclose(r.R, np.diag(scales), rtol=0, atol=50 * U * 7)
    assert np.allclose(r.Q, Q0, rtol=0, atol=200 * U)


@pytest.mark.parametrize("seed", range(5))
def test_matches_householder_well_conditioned(seed):
    """R unique for full-rank X with diag(R) > 0: kappa <= 1e3, m <= 100, n <= 10."""
    rng = np.random.default_rng(seed)
    m, n = int(rng.integers(10, 101)), int(rng.integers(1, 11))
    X = synth.randsvd(m, n, 1e3, seed=seed)
    r = oracle.scqr3(X)
    assert r.status == 0
    Qh, Rh = householder_R(X)
    tol = 1e3 * n * U * np.linalg.norm(X, 2)
    assert np.max(np.abs(r.R - Rh)) <= tol
    assert np.max(np.abs(r.Q - Qh)) <= 1e3 * n * U


@pytest.mark.parametrize("m,n", [(300, 10), (1000, 50)])
@pytest.mark.parametrize("kappa", [1e8, 1e10, 1e12, 1e14])
def test_theorem_ceilings_and_target(m, n, kappa):
    """Thm. thm:maincholqr3: orth_F <= 6{mn+n(n+1)}u, resid <= 15 n^2 u; plus the
    north-star target orth, resid <= 10 n u (observed)."""
    X = synth.randsvd(m, n, kappa, seed=int(np.log10(kappa)))
    r = oracle.scqr3(X)
    assert r.status == 0
    orth = oracle.orth_F(r.Q)
    res = oracle.resid_F(X, r.Q, r.R)
    assert orth <= 6 * (m * n + n * (n + 1)) * U
    assert res * np.linalg.norm(X, "fro") / np.linalg.norm(X, 2) <= 15 * n * n * U
    assert orth <= 10 * n * U and res <= 10 * n * U
    assert np.all(np.diag(r.R) > 0) and np.array_equal(r.R, np.triu(r.R))
    assert r.trace[0].shifted
    if kappa <= 1 / U / (96 * (m * n + n * (n + 1))):   # eq. (guarantee)
        assert [t.shifted for t in r.trace] == [True, False, False]


def test_alg3_regime_is_exactly_three_passes():
    """In Alg. 3's proven regime the controller runs shifted, plain, plain."""
    X = synth.randsvd(2000, 16, 1e12, seed=0)   # PR1
    r = oracle.scqr3(X)
    assert r.status == 0 and r.passes == 3
    assert [t.shifted for t in r.trace] == [True, False, False]
    assert r.trace[0].shift == pytest.approx(oracle.shift(2000, 16, 1.0), rel=0.02)  # ||X||_2 = 1


def test_cholesky_qr2_breaks_down_where_shifted_succeeds():
    """PR1 (kappa=1e12 > u^-1/2): unshifted CholeskyQR2 breaks down."""
    broke = 0
    for seed in range(5):
        X = synth.randsvd(2000, 16, 1e12, seed=seed)
        plain = oracle.scqr3(X, shift_mode=oracle.SHIFT_NONE, max_passes=2)
        broke += plain.status == 2
        ok = oracle.scqr3(X)
        assert ok.status == 0 and oracle.orth_F(ok.Q) <= 10 * 16 * U
    assert broke == 5


def closed_form_kappa_q1(sig, s):
    """kappa_2(X R^-1) with R^T R = X^T X + sI in exact arithmetic (P:555-563 with E=0)."""
    return (sig[0] / np.sqrt(sig[0] ** 2 + s)) * (np.sqrt(sig[-1] ** 2 + s) / sig[-1])


@pytest.mark.parametrize("tab", ["table1", "table2"])
def test_paper_tables_1_2(tab):
    t = TABLES[tab]
    m, n, kappa = t["m"], t["n"], t["kappa"]
    X = synth.randsvd(m, n, kappa, seed=1)
    one = oracle.scqr3(X, max_passes=1)               # Q^(1): status 3 by construction
    kq1 = np.linalg.cond(one.Q)
    s = one.trace[0].shift
    alpha = s / np.linalg.norm(X, 2) ** 2
    # Theorem (eq. CNreduction): kappa(Q1) <= 2 sqrt(3) sqrt(1 + alpha kappa^2)
    assert kq1 <= 2 * np.sqrt(3) * np.sqrt(1 + alpha * kappa ** 2)
    # exact-arithmetic closed form and the paper's printed value, to an order of magnitude
    cf = closed_form_kappa_q1(synth.sigma(n, kappa), s)
    assert cf / 3 <= kq1 <= cf * 3
    assert t["kappa_Q"][0] / 30 <= kq1 <= t["kappa_Q"][0] * 30
    o1 = np.linalg.norm(one.Q.T @ one.Q - np.eye(n), 2)
    assert 0.1 <= o1 < 2.0                              # Lemma 1: < 2; paper prints 1.00
    full = oracle.scqr3(X)
    assert full.status == 0 and full.passes == 3
    o3 = np.linalg.norm(full.Q.T @ full.Q - np.eye(n), 2)
    assert o3 <= 30 * t["orth2"][2]


def test_oblique_identity_metric_reduces_to_standard():
    """B = I: oblique sCholQR3 is the standard one up to the shift formula."""
    X = synth.randsvd(500, 12, 1e10, seed=3)
    a = oracle.scqr3(X)
    b = oracle.scqr3(X, np.ones(500), np.zeros(500))
    assert a.status == b.status == 0
    assert np.max(np.abs(a.R - b.R)) <= 1e-13 * np.max(np.abs(a.R))


def test_oblique_diagonal_metric_closed_form():
    """B = D diagonal: the B-QR of X is the standard QR of D^1/2 X, Q_B = D^-1/2 Q."""
    X = synth.randsvd(400, 9, 1e6, seed=4)
    d = 10.0 ** np.random.default_rng(0).uniform(0, 2, 400)
    r = oracle.scqr3(X, d, np.zeros(400))
    assert r.status == 0
    Qh, Rh = householder_R(np.sqrt(d)[:, None] * X)
    assert np.max(np.abs(r.R - Rh)) <= 1e-12 * np.max(np.abs(Rh))
    assert np.max(np.abs(r.Q - Qh / np.sqrt(d)[:, None])) <= 1e-9


def test_oblique_tridiagonal_ceilings():
    """Thm. thm:Bsta on the BASELINE config-5 construction at desk size."""
    m, n = 3000, 16
    X = synth.randsvd(m, n, 1e12, seed=0)
    d, e = synth.tridiag_b(m, seed=0)
    r = oracle.scqr3(X, d, e)
    assert r.status == 0
    B = np.diag(d) + np.diag(e[:-1], 1) + np.diag(e[:-1], -1)
    ev = np.linalg.eigvalsh(B)
    kB = ev[-1] / ev[0]
    orthB = oracle.orth_F(r.Q, d, e)
    res = oracle.resid_F(X, r.Q, r.R)
    assert orthB <= 8 * (m * np.sqrt(m * n) + n * (n + 1)) * U * kB
    assert res <= 16 * n * n * U * kB ** 1.5
    assert orthB <= 10 * n * U and res <= 10 * n * U
    assert r.trace[0].shifted
    # Q is B-orthonormal, not orthonormal: guards against B being silently dropped
    assert oracle.orth_F(np.asfortranarray(r.Q)) > 1e-3


def test_rank_emulation_changes_rounding_only():
    X = synth.randsvd(5000, 24, 1e12, seed=6)
    a = oracle.scqr3(X)
    for p in (2, 3, 8):
        b = oracle.scqr3(X, nparts=p)
        assert b.status == 0
        assert np.max(np.abs(a.R - b.R)) <= 1e-10 * np.max(np.abs(a.R))


def test_near_u_inverse_needs_more_passes_and_still_converges():
    """kappa ~ 1e15 ("more shiftedCholeskyQR iterations would be needed")."""
    X = synth.randsvd(1000, 50, 1e15, seed=0)
    r = oracle.scqr3(X)
    assert r.status == 0 and r.passes >= 4
    assert oracle.orth_F(r.Q) <= 10 * 50 * U
    assert oracle.resid_F(X, r.Q, r.R) <= 10 * 50 * U


def test_status_codes():
    X = synth.randsvd(100, 5, 1e3, seed=0)
    r = oracle.scqr3(X, max_passes=1)
    assert r.status == 3 and r.passes == 1
    Z = np.zeros((50, 3))                               # rank-deficient: unsupported
    r = oracle.scqr3(Z)
    assert r.status in (2, 3)


# ------------------------------------------------ shift policies beyond Alg. 3
@pytest.mark.parametrize("kappa", [1e2, 1e5, 1e7])
def test_adaptive_is_cholesky_qr2_below_u_half(kappa):
    """Alg. 2 shifts only on breakdown: for kappa(X) < u^-1/2 no Cholesky breaks
    down and two plain passes (CholeskyQR2) give R = Householder's R."""
    X = synth.randsvd(3000, 12, kappa, seed=4)
    r = oracle.scqr3(X, shift_mode=oracle.SHIFT_ADAPTIVE)
    assert r.status == 0 and r.passes == 2
    assert not any(t.shifted for t in r.trace) and all(t.breakdown_pivot == 0 for t in r.trace)
    _, Rh = householder_R(X)
    assert np.max(np.abs(r.R - Rh)) <= 1e3 * 12 * U * kappa * np.linalg.norm(X, 2)
    assert oracle.orth_F(r.Q) <= 10 * 12 * U and oracle.resid_F(X, r.Q, r.R) <= 10 * 12 * U


def test_adaptive_shifts_after_a_pass1_breakdown():
    """PR1 (kappa=1e12): pass 1's plain Cholesky breaks down (the CholeskyQR2 failure pinned
    above), so Alg. 2 introduces the safe shift on that pass and then runs like Alg. 3."""
    X = synth.randsvd(2000, 16, 1e12, seed=0)
    r = oracle.scqr3(X, shift_mode=oracle.SHIFT_ADAPTIVE)
    plain = oracle.scqr3(X, shift_mode=oracle.SHIFT_NONE, max_passes=1)
    assert plain.status == 2
    assert r.status == 0 and r.trace[0].shifted and r.trace[0].breakdown_pivot == plain.trace[0].breakdown_pivot
    safe = oracle.scqr3(X)
    assert r.trace[0].shift == safe.trace[0].shift
    assert np.array_equal(r.R, safe.R)   # same shift on the same Gram: identical arithmetic


def test_practical_shift_first_pass_closed_form():
    """X = [diag(sigma); 0] has the exact Gram diag(sigma^2), so pass 1 of PRACTICAL gives
    R~ = diag(sqrt(sigma^2 + s)) with s = u * N^2, N^2 ~ sigma_1^2 (Remark P:1600-1606), and
    kappa(Q1) equals the closed form of P:555-563."""
    sig = np.array([1.0, 0.5, 1e-3, 2e-5, 1e-6, 3e-7])
    n = sig.size
    X = np.zeros((40, n))
    X[np.arange(n), np.arange(n)] = sig
    r = oracle.scqr3(X, shift_mode=oracle.SHIFT_PRACTICAL, max_passes=1)
    t = r.trace[0]
    assert t.shifted and t.breakdown_pivot == 0
    assert 1.0 <= t.shift / U <= 1.02     # u * 1.01 * lambda_max, lambda_max = sigma_1^2 = 1
    assert np.allclose(np.diag(r.R), np.sqrt(sig ** 2 + t.shift), rtol=4 * U, atol=0)
    kq = np.linalg.cond(r.Q)
    assert abs(kq / closed_form_kappa_q1(sig, t.shift) - 1) <= 1e-9
    safe = oracle.scqr3(X, max_passes=1)
    assert kq < np.linalg.cond(safe.Q)   # the smaller shift reduces kappa(Q1) further (Fig. 2)


def test_practical_falls_back_to_safe_shift_on_breakdown():
    """Fig. 2's setting (m=1000, n=50, kappa=1e15): chol(A + u||X||^2 I) is not guaranteed
     and breaks down here; the fallback is the safe shift (reading D21)."""
    X = synth.randsvd(1000, 50, 1e15, seed=0)
    r = oracle.scqr3(X, shift_mode=oracle.SHIFT_PRACTICAL)
    safe = oracle.scqr3(X)
    assert r.status == 0 and r.trace[0].breakdown_pivot > 0
    assert r.trace[0].shift == safe.trace[0].shift
    assert oracle.orth_F(r.Q) <= 10 * 50 * U


# ------------------------------------------------ general sparse SPD metric
def test_csr_tridiagonal_is_the_banded_method():
    """Same metric, same term order: the CSR path reproduces the pinned banded path bitwise."""
    m, n = 3000, 16
    X = synth.randsvd(m, n, 1e12, seed=0)
    d, e = synth.tridiag_b(m, seed=0)
    a = oracle.scqr3(X, d, e)
    b = oracle.scqr3(X, csr=synth.tridiag_csr(d, e))
    assert a.status == b.status == 0 and a.passes == b.passes
    assert np.array_equal(a.R, b.R) and np.array_equal(a.Q, b.Q)
    assert [t.shift for t in a.trace] == [t.shift for t in b.trace]


def test_csr_laplacian_metric_ceilings():
    """2-D Laplacian metric (stand-in for the paper's sparse SPD matrices):
    Q^T B Q = I and X = QR within Thm. thm:Bsta's ceilings, and Q is genuinely
    B-orthonormal (not orthonormal)."""
    import scipy.sparse as sp
    nx, ny, n = 60, 50, 12
    m = nx * ny
    B = synth.laplacian2d(nx, ny, seed=3, wmax=1e2)
    X = synth.randsvd(m, n, 1e10, seed=1)
    r = oracle.scqr3(X, csr=B)
    assert r.status == 0 and r.trace[0].shifted
    Bd = sp.csr_matrix((B[2], B[1], B[0]), shape=(m, m)).toarray()
    ev = np.linalg.eigvalsh(Bd)
    kB = ev[-1] / ev[0]
    orthB = oracle.orth_F_csr(r.Q, B)
    res = oracle.resid_F(X, r.Q, r.R)
    assert orthB <= 8 * (m * np.sqrt(m * n) + n * (n + 1)) * U * kB
    assert res <= 16 * n * n * U * kB ** 1.5
    assert orthB <= 10 * n * U and res <= 10 * n * U
    assert oracle.orth_F(r.Q) > 1e-3
    # brute force: Q^T B Q against the dense B in extended precision
    Ql = r.Q.astype(np.longdouble)
    G = Ql.T @ (Bd.astype(np.longdouble) @ Ql)
    assert abs(float(np.linalg.norm(G - np.eye(n), "fro")) - orthB) <= 1e-16 + 1e-3 * orthB


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_non_finite_input_is_an_invalid_argument(bad):
    """entries must be finite; status 1 before any factorisation."""
    X = synth.randsvd(200, 5, 1e3, seed=1)
    X[17, 3] = bad
    assert oracle.scqr3(X).status == 1
