"""CPU oracle for shifted CholeskyQR3 (arXiv:1809.11085) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1809_11085_b200`` never imports it and shares no code with it.

The arithmetic lives in plain C (``scqr3_oracle.c``, fp64, ``-ffp-contract=off``);
this module only builds/loads it and marshals numpy arrays.  Every function cites
the PAPER.md passage it follows in the C source.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "scqr3_oracle.c")
_LIB = os.path.join(_HERE, "liborc.so")
_lib = None

U = 2.0 ** -53  # unit roundoff

SHIFT_SAFE, SHIFT_FIXED, SHIFT_NONE, SHIFT_ADAPTIVE, SHIFT_PRACTICAL = 0, 1, 2, 3, 4
NORM_POWER, NORM_FROBENIUS, NORM_USER = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, OpenMP over independent outputs only)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


class _Opts(ctypes.Structure):
    _fields_ = [
        ("shift_mode", ctypes.c_int), ("shift_value", ctypes.c_double),
        ("norm_mode", ctypes.c_int), ("norm2_bound", ctypes.c_double),
        ("bnorm_bound", ctypes.c_double), ("max_passes", ctypes.c_int),
        ("stop_tol", ctypes.c_double), ("power_iters", ctypes.c_int),
        ("m_global", ctypes.c_double), ("nparts", ctypes.c_int),
    ]


class _Trace(ctypes.Structure):
    _fields_ = [
        ("shift", ctypes.c_double), ("shifted", ctypes.c_int),
        ("breakdown_pivot", ctypes.c_int), ("pivot_value", ctypes.c_double),
        ("norm2_est", ctypes.c_double), ("dev_F", ctypes.c_double),
    ]


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.POINTER(ctypes.c_double)
        i64, dbl = ctypes.c_int64, ctypes.c_double
        lib.orc_gram.argtypes = [i64, i64, P, i64, P]
        lib.orc_gram_oblique.argtypes = [i64, i64, P, i64, P, P, P, P]
        PI64, PI32 = ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32)
        lib.orc_gram_oblique_csr.argtypes = [i64, i64, P, i64, PI64, PI32, P, P, P]
        lib.orc_gram_parts.argtypes = [i64, i64, P, i64, P, P, PI64, PI32, P, ctypes.c_int, P, P]
        lib.orc_orth_F_csr.argtypes = [i64, i64, P, i64, PI64, PI32, P]
        lib.orc_orth_F_csr.restype = dbl
        lib.orc_scqr3_csr.argtypes = [i64, i64, P, i64, PI64, PI32, P, P, i64, P, ctypes.POINTER(_Opts),
                                      ctypes.POINTER(_Trace), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        lib.orc_scqr3_csr.restype = ctypes.c_int
        lib.orc_cholesky.argtypes = [i64, P, dbl, P, ctypes.POINTER(i64), P]
        lib.orc_cholesky.restype = ctypes.c_int
        lib.orc_trsm_rows.argtypes = [i64, i64, P, i64, P, P, i64]
        lib.orc_trmul.argtypes = [i64, P, P]
        lib.orc_power_lmax.argtypes = [i64, P, ctypes.c_int]
        lib.orc_power_lmax.restype = dbl
        lib.orc_shift.argtypes = [dbl, dbl, dbl]
        lib.orc_shift.restype = dbl
        lib.orc_shift_oblique.argtypes = [dbl, dbl, dbl, dbl]
        lib.orc_shift_oblique.restype = dbl
        lib.orc_orth_F.argtypes = [i64, i64, P, i64, P, P]
        lib.orc_orth_F.restype = dbl
        lib.orc_resid_F.argtypes = [i64, i64, P, i64, P, i64, P]
        lib.orc_resid_F.restype = dbl
        lib.orc_scqr3.argtypes = [i64, i64, P, i64, P, P, P, i64, P, ctypes.POINTER(_Opts),
                                  ctypes.POINTER(_Trace), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        lib.orc_scqr3.restype = ctypes.c_int
        lib.orc_zgram.argtypes = [i64, i64, P, i64, P]
        lib.orc_zcholesky.argtypes = [i64, P, dbl, P, ctypes.POINTER(i64), P]
        lib.orc_zcholesky.restype = ctypes.c_int
        lib.orc_ztrsm_rows.argtypes = [i64, i64, P, i64, P, P, i64]
        lib.orc_ztrmul.argtypes = [i64, P, P]
        lib.orc_zpower_lmax.argtypes = [i64, P, ctypes.c_int]
        lib.orc_zpower_lmax.restype = dbl
        lib.orc_zorth_F.argtypes = [i64, i64, P, i64]
        lib.orc_zorth_F.restype = dbl
        lib.orc_zresid_F.argtypes = [i64, i64, P, i64, P, i64, P]
        lib.orc_zresid_F.restype = dbl
        lib.orc_zscqr3.argtypes = [i64, i64, P, i64, P, i64, P, ctypes.POINTER(_Opts),
                                   ctypes.POINTER(_Trace), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        lib.orc_zscqr3.restype = ctypes.c_int
        lib.orc_num_threads.restype = ctypes.c_int
        lib.orc_set_num_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _p(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _colmajor(X: np.ndarray) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    return np.asfortranarray(X)


def num_threads() -> int:
    return _load().orc_num_threads()


def set_num_threads(t: int) -> None:
    _load().orc_set_num_threads(int(t))


def gram(X) -> np.ndarray:
    """A = X^T X, rows ascending, mirrored."""
    X = _colmajor(X)
    m, n = X.shape
    A = np.zeros((n, n), order="F")
    _load().orc_gram(m, n, _p(X), m, _p(A))
    return A


def gram_oblique(X, d, e):
    """A = X^T B X with B = tridiag(e, d, e), symmetrised; also diag(X^T X)."""
    X = _colmajor(X)
    m, n = X.shape
    d = np.ascontiguousarray(d, dtype=np.float64)
    e = np.ascontiguousarray(e, dtype=np.float64)
    A = np.zeros((n, n), order="F")
    cs = np.zeros(n)
    _load().orc_gram_oblique(m, n, _p(X), m, _p(d), _p(e), _p(A), _p(cs))
    return A, cs


def _csr(B):
    """(row_ptr int64[m+1], col_idx int32[nnz], vals float64[nnz]) -> ctypes pointers."""
    rp, ci, cv = B
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int32)
    cv = np.ascontiguousarray(cv, dtype=np.float64)
    keep = (rp, ci, cv)
    return (rp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ci.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            _p(cv), keep)


def gram_oblique_csr(X, B):
    """A = X^T B X for a CSR metric B, symmetrised; also diag(X^T X)."""
    X = _colmajor(X)
    m, n = X.shape
    prp, pci, pcv, keep = _csr(B)
    A = np.zeros((n, n), order="F")
    cs = np.zeros(n)
    _load().orc_gram_oblique_csr(m, n, _p(X), m, prp, pci, pcv, _p(A), _p(cs))
    del keep
    return A, cs


def gram_parts(X, nparts: int, d=None, e=None, csr=None):
    """The pass Gram of scqr3(..., nparts=P): contiguous row blocks' Grams summed in rank order
    (oblique: each block's X_p^T (B X)_p with the halo rows of its neighbours, symmetrised after
    the sum).  Returns (A, colsq) -- colsq (diag(X^T X)) only for an oblique metric."""
    X = _colmajor(X)
    m, n = X.shape
    A = np.zeros((n, n), order="F")
    cs = np.zeros(n)
    if d is not None:
        d = np.ascontiguousarray(d, dtype=np.float64)
        e = np.ascontiguousarray(e, dtype=np.float64)
    if csr is not None:
        prp, pci, pcv, keep = _csr(csr)
    else:
        prp = pci = pcv = keep = None
    _load().orc_gram_parts(m, n, _p(X), m, _p(d), _p(e), prp, pci, pcv, int(nparts), _p(A), _p(cs))
    del keep
    return A, cs


def orth_F_csr(Q, B) -> float:
    """||Q^T B Q - I||_F for a CSR metric, Dot2-compensated."""
    Q = _colmajor(Q)
    m, n = Q.shape
    prp, pci, pcv, keep = _csr(B)
    r = float(_load().orc_orth_F_csr(m, n, _p(Q), m, prp, pci, pcv))
    del keep
    return r


@dataclass
class Breakdown:
    pivot: int       # 1-based column of the first non-positive / non-finite pivot
    value: float     # the pivot value before the square root


def cholesky(A, s: float = 0.0):
    """R with R^T R = A + sI (unblocked right-looking), or Breakdown."""
    A = np.asfortranarray(np.asarray(A, dtype=np.float64))
    n = A.shape[0]
    R = np.zeros((n, n), order="F")
    piv = ctypes.c_int64(0)
    pv = ctypes.c_double(0)
    rc = _load().orc_cholesky(n, _p(A), float(s), _p(R), ctypes.byref(piv), ctypes.byref(pv))
    if rc:
        return Breakdown(int(piv.value), float(pv.value))
    return R


def trsm_rows(X, R) -> np.ndarray:
    """Q = X R^{-1} by row-wise forward substitution with division."""
    X = _colmajor(X)
    R = np.asfortranarray(np.asarray(R, dtype=np.float64))
    m, n = X.shape
    Q = np.zeros((m, n), order="F")
    _load().orc_trsm_rows(m, n, _p(X), m, _p(R), _p(Q), m)
    return Q


def trmul(Rt, R) -> np.ndarray:
    """Returns Rt @ R for upper-triangular factors, k ascending."""
    Rt = np.asfortranarray(np.asarray(Rt, dtype=np.float64))
    out = np.array(R, dtype=np.float64, order="F", copy=True)
    _load().orc_trmul(Rt.shape[0], _p(Rt), _p(out))
    return out


def power_lmax(A, iters: int = 32) -> float:
    """Rayleigh quotient after `iters` power steps from the all-ones vector (D2)."""
    A = np.asfortranarray(np.asarray(A, dtype=np.float64))
    return float(_load().orc_power_lmax(A.shape[0], _p(A), int(iters)))


def shift(m, n, norm2sq) -> float:
    """s = 11{mn+n(n+1)} u ||X||_2^2 (eq. finds2)."""
    return float(_load().orc_shift(float(m), float(n), float(norm2sq)))


def shift_oblique(m, n, nx2, nb) -> float:
    """s = 11{2m sqrt(mn)+n(n+1)} u ||X||_2^2 ||B||_2 (eq. finds2B)."""
    return float(_load().orc_shift_oblique(float(m), float(n), float(nx2), float(nb)))


def orth_F(Q, d=None, e=None) -> float:
    """||Q^T Q - I||_F (or ||Q^T B Q - I||_F), Dot2-compensated."""
    Q = _colmajor(Q)
    m, n = Q.shape
    if d is not None:
        d = np.ascontiguousarray(d, dtype=np.float64)
        e = np.ascontiguousarray(e, dtype=np.float64)
    return float(_load().orc_orth_F(m, n, _p(Q), m, _p(d), _p(e)))


def resid_F(X, Q, R) -> float:
    """||X - QR||_F / ||X||_F, compensated (D13)."""
    X = _colmajor(X)
    Q = _colmajor(Q)
    R = np.asfortranarray(np.asarray(R, dtype=np.float64))
    m, n = X.shape
    return float(_load().orc_resid_F(m, n, _p(X), m, _p(Q), m, _p(R)))


@dataclass
class PassTrace:
    shift: float
    shifted: bool
    breakdown_pivot: int
    pivot_value: float
    norm2_est: float
    dev_F: float


@dataclass
class Result:
    status: int
    Q: np.ndarray
    R: np.ndarray
    passes: int
    trace: list


def scqr3(X, d=None, e=None, *, shift_mode=SHIFT_SAFE, shift_value=0.0, norm_mode=NORM_POWER,
          norm2_bound=0.0, bnorm_bound=0.0, max_passes=8, stop_tol=0.5, power_iters=32,
          m_global=0, nparts=1, csr=None) -> Result:
    """Shifted CholeskyQR3 with breakdown re-shift (Alg. 3 P:698-711 + Alg. 2).

    shift_mode ADAPTIVE: Alg. 2 literally (no shift on pass 1 unless chol breaks down);
    PRACTICAL: shifted attempts try s_p = u*N2 first (Remark P:1600-1606), then the safe s.
    Oblique (d, e given, or csr=(row_ptr, col_idx, vals)): Alg. 5 with the
    B-Gram in every pass (D8)."""
    X = _colmajor(X)
    m, n = X.shape
    Q = np.zeros((m, n), order="F")
    R = np.zeros((n, n), order="F")
    if d is not None:
        d = np.ascontiguousarray(d, dtype=np.float64)
        e = np.ascontiguousarray(e, dtype=np.float64)
    o = _Opts(shift_mode, shift_value, norm_mode, norm2_bound, bnorm_bound, max_passes, stop_tol,
              power_iters, float(m_global), nparts)
    cap = max(max_passes, 1)
    tr = (_Trace * cap)()
    passes = ctypes.c_int(0)
    if csr is not None:
        prp, pci, pcv, keep = _csr(csr)
        st = _load().orc_scqr3_csr(m, n, _p(X), m, prp, pci, pcv, _p(Q), m, _p(R), ctypes.byref(o), tr, cap,
                                   ctypes.byref(passes))
        del keep
    else:
        st = _load().orc_scqr3(m, n, _p(X), m, _p(d), _p(e), _p(Q), m, _p(R), ctypes.byref(o), tr, cap,
                               ctypes.byref(passes))
    k = passes.value
    trace = [PassTrace(t.shift, bool(t.shifted), t.breakdown_pivot, t.pivot_value, t.norm2_est, t.dev_F)
             for t in list(tr)[:k]]
    return Result(int(st), Q, R, k, trace)


# --------------------------------------------------------------------------- complex (N4)
def _zcol(X) -> np.ndarray:
    X = np.asarray(X, dtype=np.complex128)
    if X.ndim == 1:
        X = X[:, None]
    return np.asfortranarray(X)


def _zp(a):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def zgram(X) -> np.ndarray:
    """A = X^H X (Hermitian), rows ascending (^T -> ^H)."""
    X = _zcol(X)
    m, n = X.shape
    A = np.zeros((n, n), dtype=np.complex128, order="F")
    _load().orc_zgram(m, n, _zp(X), m, _zp(A))
    return A


def zcholesky(A, s: float = 0.0):
    A = np.asfortranarray(np.asarray(A, dtype=np.complex128))
    n = A.shape[0]
    R = np.zeros((n, n), dtype=np.complex128, order="F")
    piv = ctypes.c_int64(0)
    pv = ctypes.c_double(0)
    rc = _load().orc_zcholesky(n, _zp(A), float(s), _zp(R), ctypes.byref(piv), ctypes.byref(pv))
    return Breakdown(int(piv.value), float(pv.value)) if rc else R


def ztrsm_rows(X, R) -> np.ndarray:
    X = _zcol(X)
    R = np.asfortranarray(np.asarray(R, dtype=np.complex128))
    m, n = X.shape
    Q = np.zeros((m, n), dtype=np.complex128, order="F")
    _load().orc_ztrsm_rows(m, n, _zp(X), m, _zp(R), _zp(Q), m)
    return Q


def ztrmul(Rt, R) -> np.ndarray:
    Rt = np.asfortranarray(np.asarray(Rt, dtype=np.complex128))
    out = np.asfortranarray(np.array(R, dtype=np.complex128))
    _load().orc_ztrmul(Rt.shape[0], _zp(Rt), _zp(out))
    return out


def zpower_lmax(A, iters: int = 32) -> float:
    A = np.asfortranarray(np.asarray(A, dtype=np.complex128))
    return float(_load().orc_zpower_lmax(A.shape[0], _zp(A), iters))


def zorth_F(Q) -> float:
    Q = _zcol(Q)
    m, n = Q.shape
    return float(_load().orc_zorth_F(m, n, _zp(Q), m))


def zresid_F(X, Q, R) -> float:
    X, Q = _zcol(X), _zcol(Q)
    R = np.asfortranarray(np.asarray(R, dtype=np.complex128))
    m, n = X.shape
    return float(_load().orc_zresid_F(m, n, _zp(X), m, _zp(Q), m, _zp(R)))


def zscqr3(X, *, shift_mode=SHIFT_SAFE, shift_value=0.0, norm_mode=NORM_POWER, norm2_bound=0.0,
           max_passes=8, stop_tol=0.5, power_iters=32, m_global=0) -> Result:
    """Shifted CholeskyQR3 of a complex X (Alg. 3 + Alg. 2 with ^T -> ^H, reading D23)."""
    X = _zcol(X)
    m, n = X.shape
    Q = np.zeros((m, n), dtype=np.complex128, order="F")
    R = np.zeros((n, n), dtype=np.complex128, order="F")
    o = _Opts(shift_mode, shift_value, norm_mode, norm2_bound, 0.0, max_passes, stop_tol, power_iters,
              float(m_global), 1)
    cap = max(max_passes, 1)
    tr = (_Trace * cap)()
    passes = ctypes.c_int(0)
    st = _load().orc_zscqr3(m, n, _zp(X), m, _zp(Q), m, _zp(R), ctypes.byref(o), tr, cap, ctypes.byref(passes))
    k = passes.value
    trace = [PassTrace(t.shift, bool(t.shifted), t.breakdown_pivot, t.pivot_value, t.norm2_est, t.dev_F)
             for t in list(tr)[:k]]
    return Result(int(st), Q, R, k, trace)
