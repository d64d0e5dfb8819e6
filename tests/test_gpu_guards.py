"""Memory-safety and race evidence without compute-sanitizer (closed on this GPU pool: runs under
it left GPUs needing a reset).  For every kernel family (the cases of tools/sanitize_cases.py):

  * out-of-bounds writes: X, Q, R, the bands and the workspace sit inside larger allocations
    whose guard regions (and the padding rows of Q when ld > m) hold a NaN bit pattern; after
    the call every guard byte must be unchanged;
  * reads of uninitialised memory: the workspace is poisoned with NaN before the call, so any
    read of a workspace entry the library did not write first would turn Q or R into NaN --
    the results must be finite and equal to those of a call on a zeroed workspace;
  * races (shared-memory hazards, mbarrier phases, TMA slot reuse, cross-rank exchanges): 6
    repeated calls, some with another factorisation running concurrently on a second stream
    (different SM interleavings), must give bit-identical Q and R.
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
gpu = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1809_11085_b200 as sq
    from paper_1809_11085_b200.dist import row_block, run_ranks

GUARD = 4096  # doubles of guard on each side
NANBITS = 0x7FF4DEADBEEF0001  # a quiet-NaN payload the library never produces


def _guarded(nelem, fill=None):
    """(buffer, view) with NaN-pattern guards around a view of nelem doubles (16-B aligned)."""
    buf = torch.empty(nelem + 2 * GUARD, dtype=torch.float64, device="cuda")
    buf.view(torch.int64).fill_(NANBITS)
    view = buf[GUARD:GUARD + nelem]
    if fill is not None:
        view.copy_(fill)
    return buf, view


def _guards_intact(buf, nelem):
    b = buf.view(torch.int64)
    return bool((b[:GUARD] == NANBITS).all()) and bool((b[GUARD + nelem:] == NANBITS).all())


def _colmajor_guarded(X, pad_rows=6):
    """X (m, n) in a guarded buffer with ld = m + pad_rows (even); the pad rows keep the NaN
    pattern and are checked too."""
    m, n = X.shape
    ld = m + pad_rows + ((m + pad_rows) % 2)
    buf, v = _guarded(ld * n)
    mat = v.view(n, ld).t()[:m]
    mat.copy_(torch.as_tensor(X, device="cuda"))
    return buf, mat, ld


def _pads_intact(mat_buf, m, n, ld):
    body = mat_buf[GUARD:GUARD + ld * n].view(torch.int64).view(n, ld)
    return bool((body[:, m:] == NANBITS).all())


def _factor(kind, X, aux, Q, R, ws, stream=None):
    kw = dict(Q=Q, R=R, ws=ws)
    if stream is not None:
        kw["stream"] = stream
    if kind == "standard":
        return sq.scqr3_factor(X, **kw)
    if kind == "oblique":
        return sq.scqr3_factor_oblique(X, aux[0], aux[1], **kw)
    return sq.scqr3_factor_oblique_csr(X, aux, **kw)


CASES = [("standard", 2000, 16, 1e12), ("standard", 40_000, 40, 1e9), ("standard", 40_000, 128, 1e10),
         ("standard", 40_000, 256, 1e8), ("standard", 40_000, 300, 1e8), ("oblique", 40_000, 64, 1e10),
         ("csr", 20_000, 32, 1e8),
         # round 2: m % 32 == 0 (32-row Gram stages through the 3-D map) with the inverse-diagonal
         # TRSM (n = 128; fused with the next Gram at n = 64), and the n = 96 inverse instance
         ("standard", 40_960, 128, 1e10), ("standard", 32_768, 64, 1e12), ("standard", 40_000, 96, 1e8)]


@gpu
@pytest.mark.parametrize("kind,m,n,kappa", CASES)
def test_guards_poison_and_repeatability(kind, m, n, kappa):
    X = synth.randsvd(m, n, kappa, seed=11)
    aux = None
    if kind == "oblique":
        d, e = synth.tridiag_b(m, seed=11)
        bd_buf, bd = _guarded(m, torch.from_numpy(d))
        be_buf, be = _guarded(m, torch.from_numpy(e))
        aux = (bd, be)
        nws = sq.workspace(m, n, oblique=True).numel() // 8
    elif kind == "csr":
        nx = 100
        B = synth.laplacian2d(nx, m // nx, seed=0, wmax=1e3)
        aux = sq.CsrMetric(*B)
        nws = sq.workspace(m, n, csr_halo=0).numel() // 8
    else:
        nws = sq.workspace(m, n).numel() // 8
    xb, Xd, ld = _colmajor_guarded(X)
    x_before = xb.clone()
    qb, Qd, ldq = _colmajor_guarded(np.zeros((m, n)))
    rb, Rv = _guarded(n * n)
    R = Rv.view(n, n).t()
    wb, wv = _guarded(nws + 32)  # (+32 doubles: slack for the 256-byte alignment of the workspace)
    off = ((256 - wv.data_ptr() % 256) % 256) // 8
    ws = wv[off:off + nws]
    ws_u8 = ws.view(torch.uint8)
    ws.view(torch.int64).fill_(NANBITS)                       # poison: uninitialised reads -> NaN
    r = _factor(kind, Xd, aux, Qd, R, ws_u8)
    torch.cuda.synchronize()
    assert r.status == 0, r.status
    Q0, R0 = Qd.clone(), R.clone()
    assert torch.isfinite(Q0).all() and torch.isfinite(R0).all()
    assert torch.equal(xb.view(torch.int64), x_before.view(torch.int64)), "X (or its padding / guards) was written"
    assert _guards_intact(qb, ldq * n) and _pads_intact(qb, m, n, ldq), "write outside Q"
    assert _guards_intact(rb, n * n), "write outside R"
    assert _guards_intact(wb, nws + 32) and bool((wv[:off].view(torch.int64) == NANBITS).all()), "write outside ws"
    if kind == "oblique":
        assert _guards_intact(bd_buf, m) and _guards_intact(be_buf, m)
    # a zeroed workspace gives the same bits (no dependence on workspace contents)
    ws.zero_()
    r = _factor(kind, Xd, aux, Qd, R, ws_u8)
    torch.cuda.synchronize()
    assert torch.equal(Qd, Q0) and torch.equal(R, R0)
    # repeatability, alone and beside a concurrent factorisation on another stream
    other = sq.to_colmajor(torch.from_numpy(synth.randsvd(60_000, 64, 1e8, seed=12)), device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ws2 = sq.workspace(60_000, 64)
    for rep in range(6):
        if rep % 2:
            with torch.cuda.stream(s2):
                sq.scqr3_factor(other, ws=ws2, stream=s2)
        with torch.cuda.stream(s1):
            r = _factor(kind, Xd, aux, Qd, R, ws_u8, stream=s1)
        torch.cuda.synchronize()
        assert r.status == 0
        assert torch.equal(Qd, Q0) and torch.equal(R, R0), f"repeat {rep} differs"


@gpu
def test_guards_loopback_ranks_repeatable():
    """Two loopback ranks (standard and tridiagonal metric): repeated multi-rank calls give the
    same bits, and no rank writes outside its Q block."""
    P, m, n = 2, 40_000, 48
    X = synth.randsvd(m, n, 1e10, seed=13)
    d, e = synth.tridiag_b(m, seed=13)
    comms = sq.Comm.loopback(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    parts = [row_block(m, r, P) for r in range(P)]
    Xs = [sq.to_colmajor(torch.from_numpy(np.asfortranarray(X[a:b])), device="cuda") for a, b in parts]
    ds = [torch.from_numpy(d[a:b].copy()).cuda() for a, b in parts]
    es = [torch.from_numpy(e[a:b].copy()).cuda() for a, b in parts]
    Qg = [_colmajor_guarded(np.zeros((b - a, n))) for a, b in parts]
    torch.cuda.synchronize()
    ref = None
    for rep in range(4):
        res = run_ranks([lambda r=r: sq.scqr3_factor_oblique(Xs[r], ds[r], es[r], Q=Qg[r][1], comm=comms[r],
                                                             stream=streams[r]) for r in range(P)])
        torch.cuda.synchronize()
        assert all(x.status == 0 for x in res)
        got = [torch.cat([g[1] for g in Qg]).clone(), res[0].R.clone()]
        if ref is None:
            ref = got
        assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1])
        for (a, b), (qb, _, ldq) in zip(parts, Qg):
            assert _guards_intact(qb, ldq * n) and _pads_intact(qb, b - a, n, ldq)
    for c in comms:
        c.destroy()


@gpu
def test_guards_host_batch():
    """scqr3_factor_host_batch on a NaN-poisoned, guarded workspace (three staging buffers plus the
    factorisation workspace): every matrix finite and equal to its own scqr3_factor_host call,
    no write outside the workspace."""
    m, n, count = 9_001, 48, 4
    Xs = [synth.randsvd(m, n, 10.0 ** (3 + 2 * i), seed=20 + i) for i in range(count)]

    def pin(A=None, shape=(m, n)):
        T = torch.empty(shape[::-1], dtype=torch.float64, pin_memory=True)
        if A is not None:
            T.copy_(torch.from_numpy(np.ascontiguousarray(A.T)))
        return T.t()

    Xh = [pin(X) for X in Xs]
    Qh = [pin() for _ in range(count)]
    Rh = [pin(shape=(n, n)) for _ in range(count)]
    nws = (sq._abi.lib().scqr3_host_batch_workspace_size(m, n) + 7) // 8
    wb, wv = _guarded(nws + 32)
    off = ((256 - wv.data_ptr() % 256) % 256) // 8
    ws = wv[off:off + nws]
    ws.view(torch.int64).fill_(NANBITS)
    st = sq.scqr3_factor_host_batch(Xh, Qh, Rh, ws=ws.view(torch.uint8))
    torch.cuda.synchronize()
    assert st == [0] * count
    assert _guards_intact(wb, nws + 32) and bool((wv[:off].view(torch.int64) == NANBITS).all()), "write outside ws"
    for i in range(count):
        assert torch.isfinite(Qh[i]).all() and torch.isfinite(Rh[i]).all()
        r1 = sq.scqr3_factor_host(Xh[i])
        assert np.array_equal(r1.R.numpy(), Rh[i].numpy()) and np.array_equal(r1.Q.numpy(), Qh[i].numpy())


@gpu
def test_guards_ghost_plan_ranks():
    """Three loopback ranks with a ghost-row CSR plan (randomly permuted 2-D Laplacian): repeated
    calls give the same bits and no rank writes outside its Q block."""
    from paper_1809_11085_b200.dist import csr_ghost_plan
    P, m, n = 3, 30_000, 32
    X = synth.randsvd(m, n, 1e8, seed=14)
    rp, ci, cv = synth.laplacian2d(150, m // 150, seed=0, wmax=1e3)
    perm = np.random.default_rng(5).permutation(m)
    inv = np.empty(m, dtype=np.int64)
    inv[perm] = np.arange(m)
    nrp = np.concatenate([[0], np.cumsum(np.diff(rp)[perm])])
    idx = np.concatenate([np.arange(rp[o], rp[o + 1]) for o in perm])
    plans = csr_ghost_plan(nrp, inv[ci[idx]], cv[idx], m, P)
    comms = sq.Comm.loopback(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    parts = [row_block(m, r, P) for r in range(P)]
    Xs = [sq.to_colmajor(torch.from_numpy(np.asfortranarray(X[a:b])), device="cuda") for a, b in parts]
    Bs = [sq.CsrMetric(pl["row_ptr"], pl["col_idx"], pl["vals"],
                       ghosts=(pl["nghost"], pl["recv_counts"], pl["send_counts"], pl["send_rows"])) for pl in plans]
    Qg = [_colmajor_guarded(np.zeros((b - a, n))) for a, b in parts]
    torch.cuda.synchronize()
    ref = None
    for rep in range(3):
        res = run_ranks([lambda r=r: sq.scqr3_factor_oblique_csr(Xs[r], Bs[r], Q=Qg[r][1], comm=comms[r],
                                                                 stream=streams[r]) for r in range(P)])
        torch.cuda.synchronize()
        assert all(x.status == 0 for x in res)
        got = [torch.cat([g[1] for g in Qg]).clone(), res[0].R.clone()]
        assert torch.isfinite(got[0]).all()
        if ref is None:
            ref = got
        assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1])
        for (a, b), (qb, _, ldq) in zip(parts, Qg):
            assert _guards_intact(qb, ldq * n) and _pads_intact(qb, b - a, n, ldq)
    for c in comms:
        c.destroy()
