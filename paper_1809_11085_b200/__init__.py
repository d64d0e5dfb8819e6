"""Shifted CholeskyQR3 (arXiv:1809.11085) on NVIDIA B200 -- thin Python binding of libscqr3.so.

Every step of the factorisation runs in the library's sm_100a kernels; this module only
marshals torch tensors (device memory, streams) into the C ABI of include/scqr3.h.  There is
no CPU fallback: if the library is missing, every call raises.

Matrices are column-major: an (m, n) torch tensor with strides (1, ld), ld even (TMA).  Use
``colmajor_empty`` / ``to_colmajor`` to make one.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

from . import _abi
from ._abi import (EBREAKDOWN, EINVAL, ENOCONV, NORM_FROBENIUS, NORM_POWER, NORM_USER, OK,  # noqa: F401
                   SHIFT_ADAPTIVE, SHIFT_FIXED, SHIFT_NONE, SHIFT_PRACTICAL, SHIFT_SAFE,
                   TRSM_DIAG_AUTO, TRSM_DIAG_INVERSE, TRSM_DIAG_SUBST)

__all__ = [
    "scqr3_factor", "scqr3_factor_oblique", "scqr3_factor_host", "scqr3_gram", "scqr3_gram_oblique",
    "scqr3_cholesky", "scqr3_trsm", "colmajor_empty", "to_colmajor", "workspace", "Comm", "Result",
    "ScqrError", "launch_count", "library_path", "CsrMetric", "scqr3_factor_oblique_csr",
    "scqr3_gram_oblique_csr", "scqr3_factor_complex", "colmajor_empty_complex", "scqr3_factor_host_batch",
]

library_path = _abi.LIB_PATH


class ScqrError(RuntimeError):
    pass


@dataclass
class Result:
    status: int
    Q: object
    R: object
    passes: int
    trace: list = field(default_factory=list)


def _torch():
    import torch

    return torch


def _check(rc: int) -> int:
    if rc == EINVAL:
        raise ScqrError(_abi.last_error())
    return rc


def even_ld(m: int) -> int:
    return max(2, (m + 1) // 2 * 2)


def colmajor_empty(m: int, n: int, device="cuda", ld: int | None = None):
    """Uninitialised (m, n) float64 tensor with column-major strides (1, ld), ld even."""
    torch = _torch()
    ld = ld or even_ld(m)
    return torch.empty((n, ld), dtype=torch.float64, device=device).t()[:m]


def to_colmajor(X, device=None):
    """Column-major float64 copy (or X itself if it already qualifies)."""
    torch = _torch()
    X = torch.as_tensor(X)
    dev = device if device is not None else X.device
    if (X.dtype == torch.float64 and X.device == torch.device(dev) and X.dim() == 2 and X.stride(0) == 1
            and X.stride(1) >= max(X.shape[0], 1) and X.stride(1) % 2 == 0 and X.data_ptr() % 16 == 0):
        return X
    out = colmajor_empty(X.shape[0], X.shape[1], device=dev)
    out.copy_(X)
    return out


def _square_colmajor(A):
    """n x n float64 CUDA matrix with leading dimension exactly n (the ABI's R / A layout)."""
    torch = _torch()
    A = torch.as_tensor(A, dtype=torch.float64)
    if not A.is_cuda:
        A = A.cuda()
    return A.t().contiguous().t()


def _ld(X) -> int:
    if X.dim() != 2 or X.stride(0) != 1:
        raise ScqrError("matrix must be column-major: an (m, n) tensor with stride (1, ld)")
    return max(X.stride(1), 1) if X.shape[1] > 1 else even_ld(X.shape[0])


def workspace(m: int, n: int, oblique: bool = False, device="cuda", host_io: bool = False, csr_halo=None):
    torch = _torch()
    L = _abi.lib()
    if csr_halo is not None:
        nbytes = L.scqr3_workspace_size_csr(m, n, int(csr_halo))
    else:
        nbytes = L.scqr3_host_workspace_size(m, n) if host_io else L.scqr3_workspace_size(m, n, int(oblique))
    if nbytes == 0:
        raise ScqrError(f"unsupported size m={m} n={n}")
    return torch.empty(nbytes, dtype=torch.uint8, device=device)


class Comm:
    """NCCL communicator of libscqr3 for one rank (one process per GPU)."""

    def __init__(self, handle, rank: int, world: int):
        self.handle, self.rank, self.world = handle, rank, world

    @classmethod
    def create(cls, group=None):
        """Collective over torch.distributed: rank 0 makes the NCCL id, everybody inits."""
        torch = _torch()
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        buf = ctypes.create_string_buffer(_abi.COMM_ID_BYTES)
        if rank == 0:
            _check(_abi.lib().scqr3_comm_unique_id(buf))
        backend = dist.get_backend(group)
        dev = "cuda" if backend == "nccl" else "cpu"
        t = torch.tensor(list(buf.raw), dtype=torch.uint8, device=dev)
        dist.broadcast(t, src=0, group=group)
        raw = bytes(t.cpu().tolist())
        h = ctypes.c_void_p()
        _check(_abi.lib().scqr3_comm_init(ctypes.byref(h), world, raw, rank))
        return cls(h, rank, world)

    @classmethod
    def loopback(cls, world: int):
        """`world` in-process ranks on the current GPU (scqr3_comm_init_loopback): rank r's
        calls must be made by a host thread of its own, concurrently with the other ranks'
        (see ``paper_1809_11085_b200.dist.run_ranks``)."""
        hs = (ctypes.c_void_p * world)()
        _check(_abi.lib().scqr3_comm_init_loopback(hs, world))
        return [cls(ctypes.c_void_p(hs[r]), r, world) for r in range(world)]

    def destroy(self):
        if self.handle:
            _abi.lib().scqr3_comm_destroy(self.handle)
            self.handle = None


def _opts(shift_mode=SHIFT_SAFE, shift_value=0.0, norm_mode=NORM_POWER, norm2_bound=0.0, bnorm_bound=0.0,
          max_passes=8, stop_tol=0.5, power_iters=32, m_global=0, stream=None, comm=None, ws=None,
          trace_cap=16, prof=None, deterministic=False, trsm_diag=0):
    torch = _torch()
    o = _abi.Opts()
    _abi.lib().scqr3_default_opts(ctypes.byref(o))
    o.shift_mode, o.shift_value = shift_mode, float(shift_value)
    o.norm_mode, o.norm2_bound, o.bnorm_bound = norm_mode, float(norm2_bound), float(bnorm_bound)
    o.max_passes, o.stop_tol, o.power_iters = int(max_passes), float(stop_tol), int(power_iters)
    o.m_global = int(m_global)
    o.deterministic = 1 if deterministic else 0
    o.trsm_diag = int(trsm_diag)  # TRSM_DIAG_AUTO / _SUBST / _INVERSE (reading D24)
    if stream is None:
        stream = torch.cuda.current_stream()
    o.stream = ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    o.comm = comm.handle if isinstance(comm, Comm) else comm
    if ws is not None:
        o.workspace, o.workspace_bytes = ctypes.c_void_p(ws.data_ptr()), ws.numel()
    tr = (_abi.PassTrace * trace_cap)()
    passes = ctypes.c_int32(0)
    o.trace = ctypes.cast(tr, ctypes.POINTER(_abi.PassTrace))
    o.trace_cap = trace_cap
    o.passes_out = ctypes.pointer(passes)
    if prof is not None:
        o.prof = ctypes.pointer(prof)
    return o, tr, passes


def _trace(tr, k):
    return [dict(shift=t.shift, shifted=bool(t.shifted), breakdown_pivot=t.breakdown_pivot,
                 pivot_value=t.pivot_value, norm2_est=t.norm2_est, dev_F=t.dev_F) for t in list(tr)[:k]]


def scqr3_factor(X, *, Q=None, R=None, ws=None, inplace=False, **kw) -> Result:
    """Shifted CholeskyQR3 of a column-major CUDA float64 X (Alg. 3 + Alg. 2 re-shift)."""
    torch = _torch()
    m, n = X.shape
    if Q is None:
        Q = X if inplace else colmajor_empty(m, n, device=X.device)
    if R is None:
        R = torch.empty((n, n), dtype=torch.float64, device=X.device).t()  # column-major n x n
    if ws is None:
        ws = workspace(m, n, device=X.device)
    o, tr, passes = _opts(ws=ws, **kw)
    rc = _check(_abi.lib().scqr3_factor(m, n, X.data_ptr(), _ld(X), Q.data_ptr(), _ld(Q), R.data_ptr(),
                                        ctypes.byref(o)))
    return Result(rc, Q, R, passes.value, _trace(tr, passes.value))


def scqr3_factor_oblique(X, d, e, *, Q=None, R=None, ws=None, inplace=False, **kw) -> Result:
    """Oblique shifted CholeskyQR3 (Alg. 5, B-Gram in all passes) for tridiagonal B=(d, e)."""
    torch = _torch()
    m, n = X.shape
    if Q is None:
        Q = X if inplace else colmajor_empty(m, n, device=X.device)
    if R is None:
        R = torch.empty((n, n), dtype=torch.float64, device=X.device).t()
    if ws is None:
        ws = workspace(m, n, oblique=True, device=X.device)
    d = d.contiguous()
    e = e.contiguous()
    o, tr, passes = _opts(ws=ws, **kw)
    rc = _check(_abi.lib().scqr3_factor_oblique(m, n, X.data_ptr(), _ld(X), d.data_ptr(), e.data_ptr(),
                                                Q.data_ptr(), _ld(Q), R.data_ptr(), ctypes.byref(o)))
    return Result(rc, Q, R, passes.value, _trace(tr, passes.value))


class CsrMetric:
    """This rank's rows of a sparse SPD metric B in CSR on the device:
    row_ptr int64[m+1], col_idx int32[nnz] relative to the rank's first row (halo rows of the
    neighbours are negative / >= m), vals float64[nnz].  With a ghost plan (`ghosts=(nghost,
    recv_counts, send_counts, send_rows)`, e.g. from dist.csr_ghost_plan) indices >= m name ghost
    rows owned by other ranks, for any sparsity pattern (include/scqr3.h, SCQR3_CSR_GHOSTS)."""

    def __init__(self, row_ptr, col_idx, vals, halo: int = 0, device="cuda", ghosts=None):
        import numpy as np
        torch = _torch()
        self.row_ptr = torch.as_tensor(row_ptr, dtype=torch.int64, device=device).contiguous()
        self.col_idx = torch.as_tensor(col_idx, dtype=torch.int32, device=device).contiguous()
        self.vals = torch.as_tensor(vals, dtype=torch.float64, device=device).contiguous()
        self.halo = int(halo)
        self.nghost, self.nsend = 0, 0
        self._recv = self._send = self._rows = None
        if ghosts is not None:
            nghost, recv, send, rows = ghosts
            self.halo = _abi.CSR_GHOSTS
            self.nghost = int(nghost)
            self._recv = np.ascontiguousarray(recv, dtype=np.int64)   # host arrays (kept alive)
            self._send = np.ascontiguousarray(send, dtype=np.int64)
            self._rows = torch.as_tensor(np.asarray(rows, dtype=np.int64), device=device).contiguous()
            self.nsend = int(self._send.sum())

    def workspace_bytes(self, m: int, n: int) -> int:
        L = _abi.lib()
        if self.halo == _abi.CSR_GHOSTS:
            return int(L.scqr3_workspace_size_csr_ghosts(m, n, self.nghost, self.nsend))
        return int(L.scqr3_workspace_size_csr(m, n, self.halo))

    def c(self):
        if self.halo != _abi.CSR_GHOSTS:
            return _abi.Csr(self.row_ptr.data_ptr(), self.col_idx.data_ptr(), self.vals.data_ptr(), self.halo)
        return _abi.Csr(self.row_ptr.data_ptr(), self.col_idx.data_ptr(), self.vals.data_ptr(), self.halo,
                        self.nghost, self._recv.ctypes.data, self._send.ctypes.data, self._rows.data_ptr())


def scqr3_factor_oblique_csr(X, B: CsrMetric, *, Q=None, R=None, ws=None, inplace=False, **kw) -> Result:
    """Oblique shifted CholeskyQR3 for a general sparse SPD metric B (CSR)."""
    torch = _torch()
    m, n = X.shape
    if Q is None:
        Q = X if inplace else colmajor_empty(m, n, device=X.device)
    if R is None:
        R = torch.empty((n, n), dtype=torch.float64, device=X.device).t()
    if ws is None:
        ws = _torch().empty(B.workspace_bytes(m, n), dtype=_torch().uint8, device=X.device)
    o, tr, passes = _opts(ws=ws, **kw)
    cb = B.c()
    rc = _check(_abi.lib().scqr3_factor_oblique_csr(m, n, X.data_ptr(), _ld(X), ctypes.byref(cb), Q.data_ptr(),
                                                    _ld(Q), R.data_ptr(), ctypes.byref(o)))
    return Result(rc, Q, R, passes.value, _trace(tr, passes.value))


def scqr3_gram_oblique_csr(X, B: CsrMetric, *, ws=None, **kw):
    torch = _torch()
    m, n = X.shape
    A = torch.empty((n, n), dtype=torch.float64, device=X.device).t()
    cs = torch.empty(1, dtype=torch.float64, device=X.device)
    ws = ws if ws is not None else workspace(m, n, device=X.device, csr_halo=0)
    o, _, _ = _opts(ws=ws, **kw)
    cb = B.c()
    _check(_abi.lib().scqr3_gram_oblique_csr(m, n, X.data_ptr(), _ld(X), ctypes.byref(cb), A.data_ptr(),
                                             cs.data_ptr(), ctypes.byref(o)))
    return A, cs


def colmajor_empty_complex(m: int, n: int, ld: int | None = None, device="cuda"):
    """Column-major complex128 (m, n) tensor (strides (1, ld))."""
    torch = _torch()
    ld = ld or m
    return torch.empty((n, ld), dtype=torch.complex128, device=device).t()[:m]


def scqr3_factor_complex(X, *, Q=None, R=None, ws=None, **kw) -> Result:
    """Shifted CholeskyQR3 of a complex column-major complex128 CUDA tensor (N4, reading D23)."""
    torch = _torch()
    if X.dtype != torch.complex128:
        raise ScqrError("scqr3_factor_complex expects complex128")
    m, n = X.shape
    if X.stride(0) != 1:
        raise ScqrError("X must be column-major")
    if Q is None:
        Q = colmajor_empty_complex(m, n, device=X.device)
    if R is None:
        R = torch.empty((n, n), dtype=torch.complex128, device=X.device).t()
    if ws is None:
        nbytes = _abi.lib().scqr3_workspace_size_complex(m, n)
        if nbytes == 0:
            raise ScqrError(f"unsupported size m={m} n={n}")
        ws = torch.empty(nbytes, dtype=torch.uint8, device=X.device)
    o, tr, passes = _opts(ws=ws, **kw)
    ldx = X.stride(1) if n > 1 else max(m, 1)
    ldq = Q.stride(1) if n > 1 else max(m, 1)
    rc = _check(_abi.lib().scqr3_factor_complex(m, n, X.data_ptr(), ldx, Q.data_ptr(), ldq, R.data_ptr(),
                                                ctypes.byref(o)))
    return Result(rc, Q, R, passes.value, _trace(tr, passes.value))


def scqr3_factor_host(X, *, Q=None, R=None, ws=None, **kw) -> Result:
    """End-to-end call on HOST (CPU, ideally pinned) column-major tensors."""
    torch = _torch()
    m, n = X.shape
    if Q is None:
        Q = torch.empty((n, m), dtype=torch.float64).t()
    if R is None:
        R = torch.empty((n, n), dtype=torch.float64).t()
    if ws is None:
        ws = workspace(m, n, host_io=True)
    o, tr, passes = _opts(ws=ws, **kw)
    rc = _check(_abi.lib().scqr3_factor_host(m, n, X.data_ptr(), max(X.stride(1), m), Q.data_ptr(),
                                             max(Q.stride(1), m), R.data_ptr(), ctypes.byref(o)))
    return Result(rc, Q, R, passes.value, _trace(tr, passes.value))


def scqr3_factor_host_batch(Xs, Qs, Rs, *, ws=None, **kw) -> list:
    """Streaming end-to-end factorisation of len(Xs) independent HOST (pinned) column-major m x n
    matrices: uploads / downloads overlap the factorisations (include/scqr3.h).  Qs, Rs: output
    host tensors, one per input (entries may repeat).  Returns the per-matrix statuses."""
    import numpy as np
    torch = _torch()
    count = len(Xs)
    if not (len(Qs) == len(Rs) == count) or count == 0:
        raise ScqrError("Xs, Qs, Rs must have the same nonzero length")
    m, n = Xs[0].shape
    if ws is None:
        ws = torch.empty(_abi.lib().scqr3_host_batch_workspace_size(m, n), dtype=torch.uint8, device="cuda")
    o, tr, passes = _opts(ws=ws, **kw)
    arr = ctypes.c_void_p * count
    xp, qp, rp = arr(*[x.data_ptr() for x in Xs]), arr(*[q.data_ptr() for q in Qs]), arr(*[r.data_ptr() for r in Rs])
    st = np.zeros(count, dtype=np.int32)
    _check(_abi.lib().scqr3_factor_host_batch(count, m, n, xp, max(Xs[0].stride(1), m), qp, max(Qs[0].stride(1), m),
                                              rp, st.ctypes.data, ctypes.byref(o)))
    return [int(v) for v in st]


def scqr3_gram(X, *, ws=None, **kw):
    torch = _torch()
    m, n = X.shape
    A = torch.empty((n, n), dtype=torch.float64, device=X.device).t()
    ws = ws if ws is not None else workspace(m, n, device=X.device)
    o, _, _ = _opts(ws=ws, **kw)
    _check(_abi.lib().scqr3_gram(m, n, X.data_ptr(), _ld(X), A.data_ptr(), ctypes.byref(o)))
    return A


def scqr3_gram_oblique(X, d, e, *, ws=None, **kw):
    torch = _torch()
    m, n = X.shape
    A = torch.empty((n, n), dtype=torch.float64, device=X.device).t()
    cs = torch.empty(1, dtype=torch.float64, device=X.device)
    ws = ws if ws is not None else workspace(m, n, oblique=True, device=X.device)
    o, _, _ = _opts(ws=ws, **kw)
    _check(_abi.lib().scqr3_gram_oblique(m, n, X.data_ptr(), _ld(X), d.contiguous().data_ptr(),
                                         e.contiguous().data_ptr(), A.data_ptr(), cs.data_ptr(),
                                         ctypes.byref(o)))
    return A, cs


def scqr3_cholesky(A, s: float = 0.0, *, ws=None, **kw):
    """R = chol(A + sI) or ('breakdown', pivot, value)."""
    torch = _torch()
    n = A.shape[0]
    A = _square_colmajor(A)
    R = torch.empty((n, n), dtype=torch.float64, device=A.device).t()
    ws = ws if ws is not None else workspace(n, n, device=A.device)
    o, _, _ = _opts(ws=ws, **kw)
    piv = ctypes.c_int32(0)
    pv = ctypes.c_double(0)
    rc = _check(_abi.lib().scqr3_cholesky(n, A.data_ptr(), float(s), R.data_ptr(), ctypes.byref(piv),
                                          ctypes.byref(pv), ctypes.byref(o)))
    if rc == EBREAKDOWN:
        return ("breakdown", piv.value, pv.value)
    return R


def scqr3_trsm(X, R, *, Q=None, ws=None, **kw):
    m, n = X.shape
    Q = Q if Q is not None else colmajor_empty(m, n, device=X.device)
    R = _square_colmajor(R)
    ws = ws if ws is not None else workspace(m, n, device=X.device)
    o, _, _ = _opts(ws=ws, **kw)
    _check(_abi.lib().scqr3_trsm(m, n, X.data_ptr(), _ld(X), R.data_ptr(), Q.data_ptr(), _ld(Q),
                                 ctypes.byref(o)))
    return Q


def launch_count(reset: bool = False) -> int:
    return int(_abi.lib().scqr3_launch_count(int(reset)))
