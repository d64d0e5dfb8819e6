"""ctypes declarations for libscqr3.so (include/scqr3.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SCQR3_LIB") or os.path.join(HERE, "libscqr3.so")

SCQR3_ABI_VERSION = 2
OK, EINVAL, EBREAKDOWN, ENOCONV = 0, 1, 2, 3
SHIFT_SAFE, SHIFT_FIXED, SHIFT_NONE, SHIFT_ADAPTIVE, SHIFT_PRACTICAL = 0, 1, 2, 3, 4
NORM_POWER, NORM_FROBENIUS, NORM_USER = 0, 1, 2
TRSM_DIAG_AUTO, TRSM_DIAG_SUBST, TRSM_DIAG_INVERSE = 0, 1, 2
CSR_GHOSTS = -1
COMM_ID_BYTES = 128

EXPORTED = [
    "scqr3_default_opts", "scqr3_workspace_size", "scqr3_factor", "scqr3_factor_oblique",
    "scqr3_host_workspace_size", "scqr3_factor_host", "scqr3_gram", "scqr3_gram_oblique",
    "scqr3_cholesky", "scqr3_trsm", "scqr3_comm_unique_id", "scqr3_comm_init",
    "scqr3_comm_destroy", "scqr3_last_error", "scqr3_launch_count", "scqr3_workspace_size_csr",
    "scqr3_factor_oblique_csr", "scqr3_gram_oblique_csr", "scqr3_workspace_size_complex",
    "scqr3_factor_complex", "scqr3_comm_init_loopback", "scqr3_workspace_size_csr_ghosts",
    "scqr3_host_batch_workspace_size", "scqr3_factor_host_batch",
]


class Csr(ctypes.Structure):
    """scqr3_csr: this rank's rows of a sparse SPD metric (device arrays)."""
    _fields_ = [
        ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p), ("vals", ctypes.c_void_p),
        ("halo", ctypes.c_int64),
        # ghost-row plan (halo == CSR_GHOSTS): nghost, host recv/send counts, device send rows
        ("nghost", ctypes.c_int64), ("recv_counts", ctypes.c_void_p), ("send_counts", ctypes.c_void_p),
        ("send_rows", ctypes.c_void_p),
    ]


class PassTrace(ctypes.Structure):
    _fields_ = [
        ("shift", ctypes.c_double), ("shifted", ctypes.c_int32),
        ("breakdown_pivot", ctypes.c_int32), ("pivot_value", ctypes.c_double),
        ("norm2_est", ctypes.c_double), ("dev_F", ctypes.c_double),
    ]


class Prof(ctypes.Structure):
    _fields_ = [
        ("gram_ms", ctypes.c_double), ("gram_launches", ctypes.c_int64),
        ("reduce_ms", ctypes.c_double), ("reduce_launches", ctypes.c_int64),
        ("chol_ms", ctypes.c_double), ("chol_launches", ctypes.c_int64),
        ("trsm_ms", ctypes.c_double), ("trsm_launches", ctypes.c_int64),
        ("comm_ms", ctypes.c_double), ("comm_calls", ctypes.c_int64),
        ("trmul_ms", ctypes.c_double), ("trmul_launches", ctypes.c_int64),
    ]


class Opts(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32), ("shift_mode", ctypes.c_int32),
        ("shift_value", ctypes.c_double), ("norm_mode", ctypes.c_int32),
        ("power_iters", ctypes.c_int32), ("norm2_bound", ctypes.c_double),
        ("bnorm_bound", ctypes.c_double), ("max_passes", ctypes.c_int32),
        ("deterministic", ctypes.c_int32), ("stop_tol", ctypes.c_double),
        ("m_global", ctypes.c_int64), ("stream", ctypes.c_void_p), ("comm", ctypes.c_void_p),
        ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
        ("trace", ctypes.POINTER(PassTrace)), ("trace_cap", ctypes.c_int32),
        ("passes_out", ctypes.POINTER(ctypes.c_int32)), ("prof", ctypes.POINTER(Prof)),
        ("trsm_diag", ctypes.c_int32),
    ]


_lib = None


def lib():
    """Load libscqr3.so; fails loudly (no fallback of any kind) if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built: run `python -m paper_1809_11085_b200.build` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        i64, vp, P = ctypes.c_int64, ctypes.c_void_p, ctypes.POINTER(Opts)
        L.scqr3_default_opts.argtypes = [P]
        L.scqr3_default_opts.restype = None
        L.scqr3_workspace_size.argtypes = [i64, i64, ctypes.c_int32]
        L.scqr3_workspace_size.restype = ctypes.c_size_t
        L.scqr3_factor.argtypes = [i64, i64, vp, i64, vp, i64, vp, P]
        L.scqr3_factor_oblique.argtypes = [i64, i64, vp, i64, vp, vp, vp, i64, vp, P]
        L.scqr3_host_workspace_size.argtypes = [i64, i64]
        L.scqr3_host_workspace_size.restype = ctypes.c_size_t
        L.scqr3_factor_host.argtypes = [i64, i64, vp, i64, vp, i64, vp, P]
        L.scqr3_host_batch_workspace_size.argtypes = [i64, i64]
        L.scqr3_host_batch_workspace_size.restype = ctypes.c_size_t
        L.scqr3_factor_host_batch.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, vp, P]
        L.scqr3_gram.argtypes = [i64, i64, vp, i64, vp, P]
        L.scqr3_gram_oblique.argtypes = [i64, i64, vp, i64, vp, vp, vp, vp, P]
        PC = ctypes.POINTER(Csr)
        L.scqr3_workspace_size_csr.argtypes = [i64, i64, i64]
        L.scqr3_workspace_size_csr.restype = ctypes.c_size_t
        L.scqr3_workspace_size_csr_ghosts.argtypes = [i64, i64, i64, i64]
        L.scqr3_workspace_size_csr_ghosts.restype = ctypes.c_size_t
        L.scqr3_factor_oblique_csr.argtypes = [i64, i64, vp, i64, PC, vp, i64, vp, P]
        L.scqr3_gram_oblique_csr.argtypes = [i64, i64, vp, i64, PC, vp, vp, P]
        L.scqr3_workspace_size_complex.argtypes = [i64, i64]
        L.scqr3_workspace_size_complex.restype = ctypes.c_size_t
        L.scqr3_factor_complex.argtypes = [i64, i64, vp, i64, vp, i64, vp, P]
        L.scqr3_cholesky.argtypes = [i64, vp, ctypes.c_double, vp, ctypes.POINTER(ctypes.c_int32),
                                     ctypes.POINTER(ctypes.c_double), P]
        L.scqr3_trsm.argtypes = [i64, i64, vp, i64, vp, vp, i64, P]
        L.scqr3_comm_unique_id.argtypes = [vp]
        L.scqr3_comm_init.argtypes = [ctypes.POINTER(vp), ctypes.c_int32, vp, ctypes.c_int32]
        L.scqr3_comm_destroy.argtypes = [vp]
        L.scqr3_comm_init_loopback.argtypes = [ctypes.POINTER(vp), ctypes.c_int32]
        L.scqr3_last_error.restype = ctypes.c_char_p
        L.scqr3_launch_count.argtypes = [ctypes.c_int32]
        L.scqr3_launch_count.restype = ctypes.c_int64
        for name in ("scqr3_factor_oblique_csr", "scqr3_gram_oblique_csr", "scqr3_factor_complex",
                     "scqr3_factor", "scqr3_factor_oblique", "scqr3_factor_host", "scqr3_gram",
                     "scqr3_gram_oblique", "scqr3_cholesky", "scqr3_trsm", "scqr3_comm_unique_id",
                     "scqr3_comm_init", "scqr3_comm_destroy", "scqr3_comm_init_loopback"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def last_error() -> str:
    return lib().scqr3_last_error().decode()
