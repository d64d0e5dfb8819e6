"""Oracle pins added in round 2 (-m "not gpu"): each pins an oracle function to something other
than itself -- a value the paper prints, exact integer arithmetic, or a naive re-derivation
from the definition.

  * Table 3 (PAPER.md P:1532-1538 setup, values P:1571-1597, tab:itecholB): oblique shifted
    CholeskyQR3 with a dense SPD B = U Sigma_B U^T, kappa_2(B) = 1e8, m = 300, n = 30,
    kappa_2(X) = 1e12, through the oracle's CSR path (B written out as a dense CSR matrix).
  * orc_zorth_F / orc_zresid_F (the complex checkers behind the N4 parity claims) on
    Gaussian-integer matrices whose Q^H Q - I and X - QR are known exactly.
  * orc_gram_parts (the P-rank Gram emulation behind oracle.scqr3(nparts=P), which the
    multi-rank GPU tests compare against): exact integer X^T X and X^T B X for every split.
  * orc_gram's row blocking: bitwise equal to the plain rows-ascending loop at m > 512.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth

U = 2.0 ** -53
TABLES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables.json")))


def _dense_csr(B):
    m = B.shape[0]
    rp = np.arange(0, m * m + 1, m, dtype=np.int64)
    ci = np.tile(np.arange(m, dtype=np.int32), m)
    return rp, ci, np.ascontiguousarray(B, dtype=np.float64).reshape(-1).copy()


def _b_measure(Q, B):
    """||Q||_2 sqrt(||B||_2) / sqrt(sigma_n(Q^T B Q)): the quantity Table 3 tracks."""
    G = Q.T @ B @ Q
    lam = np.linalg.eigvalsh((G + G.T) / 2)[0]
    return np.linalg.norm(Q, 2) * np.sqrt(np.linalg.norm(B, 2)) / np.sqrt(lam)


def test_table3_oblique_dense_metric():
    t = TABLES["table3"]
    m, n = t["m"], t["n"]
    X = synth.randsvd(m, n, t["kappa_X"], seed=0)
    # B = U Sigma_B U^T with geometric Sigma_B, kappa_2(B) = 1e8, ||B||_2 = 1
    rng = np.random.default_rng([0, 11])
    Ub, _ = np.linalg.qr(rng.standard_normal((m, m)))
    sb = t["kappa_B"] ** (-np.arange(m) / (m - 1))
    B = (Ub * sb) @ Ub.T
    B = (B + B.T) / 2
    csr = _dense_csr(B)
    # Alg. 5's shift with the exact norms ||X||_2 = ||B||_2 = 1 (eq. finds2B)
    kw = dict(csr=csr, norm_mode=oracle.NORM_USER, norm2_bound=1.0, bnorm_bound=1.0)
    meas, orth2 = [], []
    for k in (1, 2, 3):
        r = oracle.scqr3(X, max_passes=k, **kw)
        assert r.passes == k
        meas.append(_b_measure(r.Q, B))
        orth2.append(np.linalg.norm(r.Q.T @ B @ r.Q - np.eye(n), 2))
    assert r.status == 0 and [p.shifted for p in r.trace] == [True, False, False]
    # pass 1: the measure drops from ~1e10 to O(sqrt(alpha kappa(B))) ~ 1e8 (printed 4.11e8) and
    # Q1^T B Q1 is far from I (printed 1.00)
    assert t["b_measure"][0] / 30 <= meas[0] <= t["b_measure"][0] * 30, meas
    assert 0.5 <= orth2[0] <= 1.5, orth2
    # passes 2-3: the measure settles at O(10) (printed 13.50 twice), below sqrt(kappa(B)) = 1e4
    for k in (1, 2):
        assert t["b_measure"][k] / 30 <= meas[k] <= t["b_measure"][k] * 30, meas
    assert abs(meas[2] / meas[1] - 1) < 0.1
    # pass 2 leaves O(1e-3 .. 1e-1) (printed 8.31e-3); pass 3 reaches rounding level (3.49e-15)
    assert 1e-5 <= orth2[1] <= 0.5, orth2
    assert orth2[2] <= 1e-13, orth2
    # the oblique ceiling of Thm. thm:Bsta
    assert orth2[2] <= 8 * (m * math.sqrt(m * n) + n * (n + 1)) * U
    # default options (power / Gershgorin norm estimates): also three passes and 10 n u
    rd = oracle.scqr3(X, csr=csr)
    assert rd.status == 0 and rd.passes == 3
    assert oracle.orth_F_csr(rd.Q, csr) <= 10 * n * U


# ------------------------------------------------------------------ complex checkers
def test_zorth_exact_gaussian_integers():
    """||Q^H Q - I||_F for a Gaussian-integer Q: Q^H Q - I is an exact integer matrix, so the
    result is sqrt of an exact integer.  Q^T Q (no conjugate) or a sign slip in the imaginary
    part gives a different value."""
    rng = np.random.default_rng(3)
    Qi = rng.integers(-3, 4, (40, 5)) + 1j * rng.integers(-3, 4, (40, 5))
    G = Qi.conj().T @ Qi - np.eye(5)        # exact in complex integers (int64 parts)
    ref = math.sqrt(int(np.sum(np.abs(G.real).astype(np.int64) ** 2 + np.abs(G.imag).astype(np.int64) ** 2)))
    assert oracle.zorth_F(Qi.astype(np.complex128)) == pytest.approx(ref, rel=4 * U)
    # a unitary-column Q with imaginary entries: exactly 0; its transpose-only Gram would be -1
    Qu = np.zeros((3, 2), dtype=np.complex128)
    Qu[0, 0], Qu[1, 1] = 1j, -1j
    assert oracle.zorth_F(Qu) == 0.0
    Qs = Qu.copy()
    Qs[2, 0] = 1j                             # column 0 now has norm^2 2: (Q^H Q - I)_00 = 1
    assert oracle.zorth_F(Qs) == 1.0
    Qc2 = np.array([[1j], [1j]])              # q^H q = 2 -> |2 - 1| = 1; q^T q = -2 would give 3
    assert oracle.zorth_F(Qc2) == 1.0


def test_zresid_exact_cases():
    """||X - QR||_F / ||X||_F: 0 for an exactly representable complex QR with imaginary parts in
    both factors (a sign slip in Im(Q) Im(R) or a conjugated R would leave a residual), and the
    exact ratio for a one-entry perturbation."""
    Q = np.zeros((4, 2), dtype=np.complex128)
    Q[0, 0], Q[1, 1] = 1j, 1.0
    R = np.array([[2.0, 1 - 1j], [0.0, 3.0 + 0j]])
    X = Q @ R                                  # exact: entries are small Gaussian integers
    assert oracle.zresid_F(X, Q, R) == 0.0
    nx2 = float(np.sum(np.abs(X) ** 2))        # exact integer
    Xp = X.copy()
    Xp[2, 1] += 2.0 ** -20 * 1j
    got = oracle.zresid_F(Xp, Q, R)
    ref = 2.0 ** -20 / math.sqrt(nx2 + 2.0 ** -40)
    assert got == pytest.approx(ref, rel=4 * U)
    Xw = Q @ R.conj()                          # the product with a conjugated R is another matrix
    assert oracle.zresid_F(Xw, Q, R) > 0.1


# ------------------------------------------------------------------ P-rank Gram emulation
@pytest.mark.parametrize("nparts", [1, 2, 3, 8])
def test_gram_parts_exact_integer(nparts):
    rng = np.random.default_rng(nparts)
    m, n = 997, 9
    X = rng.integers(-20, 21, (m, n)).astype(float)
    Xi = X.astype(np.int64)
    A, _ = oracle.gram_parts(X, nparts)
    assert np.array_equal(A, (Xi.T @ Xi).astype(float))
    # tridiagonal metric: shard products with halo rows sum to the global X^T B X exactly
    d = rng.integers(5, 50, m).astype(float)
    e = np.zeros(m)
    e[:-1] = rng.integers(-2, 3, m - 1)
    Bi = np.diag(d.astype(np.int64)) + np.diag(e[:-1].astype(np.int64), 1) + np.diag(e[:-1].astype(np.int64), -1)
    Ao, cs = oracle.gram_parts(X, nparts, d=d, e=e)
    assert np.array_equal(Ao, (Xi.T @ Bi @ Xi).astype(float))
    assert np.array_equal(cs, np.sum(Xi * Xi, axis=0).astype(float))
    # CSR metric (integer 2-D Laplacian, halo = grid width across the splits)
    L = synth.laplacian2d(997, 1)
    Ac, _ = oracle.gram_parts(X, nparts, csr=L)
    rp, ci, cv = L
    Ld = np.zeros((m, m), dtype=np.int64)
    for i in range(m):
        for z in range(rp[i], rp[i + 1]):
            Ld[i, ci[z]] = int(cv[z])
    assert np.array_equal(Ac, (Xi.T @ Ld @ Xi).astype(float))


def test_gram_parts_equals_global_gram_to_rounding():
    """Floating data: the P-part sum differs from the rows-ascending global Gram only by the
    summation order (T1 bound)."""
    X = synth.random_rows(3001, 12, seed=4)
    d, e = synth.tridiag_b(3001, seed=4)
    A4, _ = oracle.gram_parts(X, 4, d=d, e=e)
    Ag, _ = oracle.gram_oblique(X, d, e)
    Bab = np.abs(d)[:, None] * np.abs(X)
    Bab[1:] += np.abs(e[:-1])[:, None] * np.abs(X[:-1])
    Bab[:-1] += np.abs(e[:-1])[:, None] * np.abs(X[1:])
    bound = 4 * 3001 * U * (np.abs(X).T @ Bab)
    assert np.all(np.abs(A4 - Ag) <= bound)


# ------------------------------------------------------------------ Gram row blocking
def test_orc_gram_blocking_is_the_plain_loop():
    """orc_gram walks rows in blocks of 512 for locality; each entry must still be the plain
    rows-ascending sum s = s + x_ij x_il: bitwise equal to a Python loop at m = 1500."""
    m, n = 1500, 4
    X = synth.random_rows(m, n, seed=12)
    A = oracle.gram(X)
    for j in range(n):
        for l in range(n):
            s = 0.0
            xj, xl = X[:, j].tolist(), X[:, l].tolist()
            for i in range(m):
                s = s + xj[i] * xl[i]
            assert A[j, l] == s, (j, l)
