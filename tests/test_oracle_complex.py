"""Pins for the complex oracle ("everything carries over to complex
matrices", reading D23).  Independent references: the real oracle (a real input must give
the real results bit for bit -- the complex arithmetic is written out in the real order),
exact Gaussian-integer arithmetic, numpy's complex Householder QR and eigvalsh, and the
accuracy target / breakdown behaviour pinned for the real method."""
import numpy as np
import pytest

import oracle
import synth

U = 2.0 ** -53


def gint(rng, shape, lo=-9, hi=10):
    return rng.integers(lo, hi, size=shape) + 1j * rng.integers(lo, hi, size=shape)


def test_real_input_reproduces_the_real_oracle_bitwise():
    X = synth.randsvd(700, 12, 1e10, seed=2)
    Z = X.astype(np.complex128)
    assert np.array_equal(oracle.zgram(Z).real, oracle.gram(X)) and not oracle.zgram(Z).imag.any()
    A = oracle.gram(X)
    s = oracle.shift(700, 12, oracle.power_lmax(A) * 1.01)
    Rr, Rz = oracle.cholesky(A, s), oracle.zcholesky(A.astype(complex), s)
    assert np.array_equal(Rz.real, Rr) and not Rz.imag.any()
    assert np.array_equal(oracle.ztrsm_rows(Z, Rz).real, oracle.trsm_rows(X, Rr))
    assert oracle.zpower_lmax(A.astype(complex)) == oracle.power_lmax(A)
    a, b = oracle.scqr3(X), oracle.zscqr3(Z)
    assert a.passes == b.passes and np.array_equal(b.R.real, a.R) and np.array_equal(b.Q.real, a.Q)


@pytest.mark.parametrize("m,n", [(1, 1), (9, 4), (120, 7)])
def test_zgram_exact_gaussian_integers(m, n):
    rng = np.random.default_rng(m + n)
    Xi = gint(rng, (m, n))
    ref = Xi.conj().T @ Xi  # exact in complex128 for these magnitudes (integers < 2^53)
    A = oracle.zgram(Xi)
    assert np.array_equal(A, ref)
    assert np.array_equal(A, A.conj().T) and not np.diag(A).imag.any()


@pytest.mark.parametrize("n", [1, 3, 8, 20])
def test_zcholesky_recovers_integer_factor_exactly(n):
    rng = np.random.default_rng(n)
    R = np.triu(gint(rng, (n, n), -3, 4)).astype(np.complex128)
    R[np.diag_indices(n)] = 2.0 ** rng.integers(0, 3, size=n)
    A = R.conj().T @ R
    Rz = oracle.zcholesky(A)
    assert np.array_equal(Rz, R)
    bad = oracle.zcholesky(np.array([[1, 1j], [-1j, 1]], dtype=complex))  # singular Hermitian
    assert isinstance(bad, oracle.Breakdown) and bad.pivot == 2


def test_ztrsm_and_ztrmul_exact():
    rng = np.random.default_rng(7)
    m, n = 200, 9
    Q = gint(rng, (m, n)).astype(np.complex128)
    R = np.triu(gint(rng, (n, n), -3, 4)).astype(np.complex128)
    R[np.diag_indices(n)] = 2.0 ** rng.integers(0, 3, size=n)
    assert np.array_equal(oracle.ztrsm_rows(Q @ R, R), Q)
    R2 = np.triu(gint(rng, (n, n), -3, 4)).astype(np.complex128)
    assert np.array_equal(oracle.ztrmul(R, R2), R @ R2)


def test_zpower_lmax_closed_forms():
    d = np.array([3.0, 1.0, 0.5, 0.25])
    assert abs(oracle.zpower_lmax(np.diag(d).astype(complex), 64) - 3.0) <= 1e-12
    v = np.array([1, 1j, -2, 0.5 - 1j])
    A = np.outer(v, v.conj())  # rank one: lambda = |v|^2
    assert abs(oracle.zpower_lmax(A) - np.vdot(v, v).real) <= 1e-12 * np.vdot(v, v).real


@pytest.mark.parametrize("seed", range(3))
def test_zscqr3_matches_householder(seed):
    """R is unique with a real positive diagonal: numpy's complex QR, phase-normalised."""
    m, n = 80, 6
    X = synth.randsvd_complex(m, n, 1e3, seed=seed)
    r = oracle.zscqr3(X)
    assert r.status == 0
    Qh, Rh = np.linalg.qr(X)
    ph = np.diag(Rh) / np.abs(np.diag(Rh))
    Rh = Rh / ph[:, None]
    assert np.max(np.abs(r.R - Rh)) <= 1e3 * n * U * np.linalg.norm(X, 2)
    assert np.all(np.diag(r.R).imag == 0) and np.all(np.diag(r.R).real > 0)


def test_zscqr3_target_and_cholqr2_breakdown():
    """kappa = 1e12 > u^-1/2: plain CholeskyQR2 breaks down (as for real X) and the
    shifted method reaches the BJ target in Alg. 3's three passes."""
    X = synth.randsvd_complex(2000, 16, 1e12, seed=0)
    plain = oracle.zscqr3(X, shift_mode=oracle.SHIFT_NONE, max_passes=2)
    assert plain.status == 2
    r = oracle.zscqr3(X)
    assert r.status == 0 and [t.shifted for t in r.trace] == [True, False, False]
    assert oracle.zorth_F(r.Q) <= 10 * 16 * U and oracle.zresid_F(X, r.Q, r.R) <= 10 * 16 * U


def test_zscqr3_non_finite_is_invalid():
    X = synth.randsvd_complex(100, 4, 10.0, seed=1)
    X[5, 2] = complex(np.nan, 0)
    assert oracle.zscqr3(X).status == 1
