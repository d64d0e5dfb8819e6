"""libscqr3's own multi-rank code at P = 2, 4, 8 on one GPU (loopback communicator).

The method's one exchange is the sum of the per-rank Grams ("the reduction operator is
addition", Sec. 1); the oblique variant also needs each neighbour's boundary
rows of Q for Y = BQ.  Here P ranks of the library run as P host threads, each on
its own stream and row block, exchanging through scqr3_comm_init_loopback (the same protocol
and code paths as NCCL: halo branches, e_prev coupling, global m, rank-ordered Gram sum).
Each case checks:
  * every rank returns the same status, pass count and bitwise-identical R;
  * R matches oracle.scqr3(..., nparts=P) -- the oracle's P-part emulation, shard Grams summed
    in rank order -- to 1e-10 max|R| (reading D14);
  * the stitched Q meets orthogonality and residual <= 10 n u (BASELINE north_star; oracle's
    Dot2 metrics).
"""
import functools

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
gpu = pytest.mark.gpu
U = 2.0 ** -53

if torch.cuda.is_available():
    import paper_1809_11085_b200 as sq
    from paper_1809_11085_b200.dist import csr_ghost_plan, row_block, run_ranks

M, N, KAPPA = 200_000, 128, 1e10
LAP_NX = 500  # 2-D Laplacian grid width = CSR halo rows


def _permuted(B, seed=3):
    """P^T B P for a random permutation: the same SPD Laplacian with its rows and columns
    scattered, so every row's neighbours live on arbitrary ranks (no band: ghost-row plan)."""
    rp, ci, cv = B
    m = len(rp) - 1
    perm = np.random.default_rng(seed).permutation(m)      # new row i = old row perm[i]
    inv = np.empty(m, dtype=np.int64)
    inv[perm] = np.arange(m)
    cnt = rp[1:] - rp[:-1]
    nrp = np.zeros(m + 1, dtype=np.int64)
    nrp[1:] = np.cumsum(cnt[perm])
    idx = np.concatenate([np.arange(rp[o], rp[o + 1]) for o in perm])
    return nrp, inv[ci[idx]].astype(np.int32), cv[idx].copy()


@functools.lru_cache(maxsize=None)
def _inputs(kind):
    X = synth.randsvd(M, N, KAPPA, seed=0)
    if kind == "standard":
        return X, None
    if kind == "tridiag":
        return X, synth.tridiag_b(M, seed=0)
    lap = synth.laplacian2d(LAP_NX, M // LAP_NX, seed=0, wmax=1e4)
    return X, (_permuted(lap) if kind == "csr_ghost" else lap)


@functools.lru_cache(maxsize=None)
def _oracle(kind, P):
    X, B = _inputs(kind)
    if kind == "standard":
        return oracle.scqr3(X, nparts=P)
    if kind == "tridiag":
        return oracle.scqr3(X, B[0], B[1], nparts=P)
    return oracle.scqr3(X, csr=B, nparts=P)


@functools.lru_cache(maxsize=None)
def _plans(P):
    X, B = _inputs("csr_ghost")
    return csr_ghost_plan(*B, X.shape[0], P)


def _run(kind, P, deterministic, bounds=None, comms=None):
    """Factor the kind's input over P loopback ranks; returns (results, stitched Q, comms)."""
    X, B = _inputs(kind)
    m, n = X.shape
    bounds = bounds or [row_block(m, r, P) for r in range(P)]
    own = comms is None
    comms = comms or sq.Comm.loopback(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    args = []
    for r, (r0, r1) in enumerate(bounds):
        mr = r1 - r0
        Xr = sq.to_colmajor(torch.from_numpy(np.asfortranarray(X[r0:r1])), device="cuda")
        Qr = sq.colmajor_empty(mr, n)
        Rr = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
        kw = dict(Q=Qr, R=Rr, comm=comms[r], stream=streams[r], deterministic=deterministic)
        if kind == "standard":
            kw["ws"] = sq.workspace(mr, n)
            args.append((sq.scqr3_factor, (Xr,), kw))
        elif kind == "tridiag":
            d = torch.from_numpy(B[0][r0:r1].copy()).cuda()
            e = torch.from_numpy(B[1][r0:r1].copy()).cuda()
            kw["ws"] = sq.workspace(mr, n, oblique=True)
            args.append((sq.scqr3_factor_oblique, (Xr, d, e), kw))
        elif kind == "csr_ghost":
            pl = _plans(P)[r]
            csr = sq.CsrMetric(pl["row_ptr"], pl["col_idx"], pl["vals"],
                               ghosts=(pl["nghost"], pl["recv_counts"], pl["send_counts"], pl["send_rows"]))
            args.append((sq.scqr3_factor_oblique_csr, (Xr, csr), kw))
        else:
            csr = sq.CsrMetric(*synth.csr_rows(B, r0, r1), halo=LAP_NX)
            kw["ws"] = sq.workspace(mr, n, csr_halo=LAP_NX)
            args.append((sq.scqr3_factor_oblique_csr, (Xr, csr), kw))
    torch.cuda.synchronize()
    try:
        res = run_ranks([lambda f=f, a=a, kw=kw: f(*a, **kw) for f, a, kw in args])
    finally:
        if own:
            for c in comms:
                c.destroy()
    torch.cuda.synchronize()
    Q = np.concatenate([r.Q.cpu().numpy() for r in res], axis=0) if res else None
    return res, Q


def _check(kind, P, res, Q):
    X, B = _inputs(kind)
    n = X.shape[1]
    ro = _oracle(kind, P)
    assert ro.status == 0
    st = {r.status for r in res}
    assert st == {0}, st
    assert len({r.passes for r in res}) == 1
    R0 = res[0].R.cpu().numpy()
    for r in res[1:]:
        assert np.array_equal(r.R.cpu().numpy(), R0), "R differs between ranks"
    err = np.max(np.abs(R0 - ro.R)) / np.max(np.abs(ro.R))
    assert err <= 1e-10, (err, res[0].passes, ro.passes)
    if kind == "standard":
        orth = oracle.orth_F(Q)
    elif kind == "tridiag":
        orth = oracle.orth_F(Q, B[0], B[1])
    else:
        orth = oracle.orth_F_csr(Q, B)   # (csr_ghost: the permuted global B)
    resid = oracle.resid_F(X, Q, R0)
    assert orth <= 10 * n * U and resid <= 10 * n * U, (orth, resid)
    return err


@gpu
@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("kind", ["standard", "tridiag", "csr", "csr_ghost"])
@pytest.mark.parametrize("deterministic", [False, True])
def test_loopback_factor_parity(kind, P, deterministic):
    res, Q = _run(kind, P, deterministic)
    _check(kind, P, res, Q)


@gpu
def test_loopback_r_matches_one_rank_structure():
    """P ranks and one rank factor the same X: R agrees to rounding (different sum trees)."""
    X, _ = _inputs("standard")
    one = sq.scqr3_factor(sq.to_colmajor(torch.from_numpy(X), device="cuda"))
    res, _ = _run("standard", 4, False)
    R1, R4 = one.R.cpu().numpy(), res[0].R.cpu().numpy()
    assert np.max(np.abs(R1 - R4)) <= 1e-10 * np.max(np.abs(R1))


@gpu
def test_loopback_empty_rank_standard():
    """A rank with m = 0 contributes a zero Gram: the result equals the two-part emulation."""
    X, _ = _inputs("standard")
    h = M // 2
    res, Q = _run("standard", 3, False, bounds=[(0, h), (h, h), (h, M)])
    ro = _oracle("standard", 2)
    R0 = res[0].R.cpu().numpy()
    assert all(r.status == 0 for r in res)
    assert all(np.array_equal(r.R.cpu().numpy(), R0) for r in res)
    assert np.max(np.abs(R0 - ro.R)) <= 1e-10 * np.max(np.abs(ro.R))
    assert oracle.orth_F(Q) <= 10 * N * U


@gpu
def test_loopback_rejects_together():
    """Bad arguments on one rank: every rank returns SCQR3_EINVAL before any exchange; the
    group stays usable afterwards."""
    P = 3
    comms = sq.Comm.loopback(P)
    m, n = 3000, 16
    Xs = [sq.to_colmajor(torch.from_numpy(synth.random_rows(m, n, seed=r)), device="cuda") for r in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]

    def call(r, bad):
        kw = dict(comm=comms[r], stream=streams[r])
        if bad and r == 1:
            kw["max_passes"] = 99  # > the status slots: rejected locally
        try:
            return sq.scqr3_factor(Xs[r], **kw).status
        except sq.ScqrError as e:
            return str(e)

    out = run_ranks([lambda r=r: call(r, True) for r in range(P)])
    assert all(isinstance(o, str) for o in out), out
    assert "max_passes" in out[1] and "rank 1" in out[0] and "rank 1" in out[2]
    out = run_ranks([lambda r=r: call(r, False) for r in range(P)])
    assert out == [0, 0, 0]
    for c in comms:
        c.destroy()


@gpu
def test_loopback_oblique_short_rank_rejected():
    """An oblique factorisation whose middle rank owns fewer rows than the halo: all ranks
    return SCQR3_EINVAL (the neighbours would otherwise read rows that do not exist)."""
    X, B = _inputs("csr")
    bounds = [(0, 20_000), (20_000, 20_100), (20_100, 40_000)]  # 100 < LAP_NX = 500 rows
    Xs = X[:40_000]
    comms = sq.Comm.loopback(3)
    streams = [torch.cuda.Stream() for _ in range(3)]
    Bsub = synth.laplacian2d(LAP_NX, 40_000 // LAP_NX, seed=0, wmax=1e4)

    def call(r):
        r0, r1 = bounds[r]
        Xr = sq.to_colmajor(torch.from_numpy(np.asfortranarray(Xs[r0:r1])), device="cuda")
        csr = sq.CsrMetric(*synth.csr_rows(Bsub, r0, r1), halo=LAP_NX)
        try:
            return sq.scqr3_factor_oblique_csr(Xr, csr, comm=comms[r], stream=streams[r]).status
        except sq.ScqrError as e:
            return str(e)

    out = run_ranks([lambda r=r: call(r) for r in range(3)])
    assert all(isinstance(o, str) for o in out), out
    for c in comms:
        c.destroy()


@gpu
def test_loopback_csr_index_past_last_rank_rejected():
    """a CSR column index >= m on the LAST rank (no next rank to supply halo rows)
    is an invalid argument on every rank."""
    m, n = 4000, 8
    P = 2
    comms = sq.Comm.loopback(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    rp = np.arange(m + 1, dtype=np.int64)
    vals = np.ones(m)

    def call(r):
        ci = np.arange(m, dtype=np.int32)
        if r == P - 1:
            ci[-1] = m  # would be the next rank's first row
        Xr = sq.to_colmajor(torch.from_numpy(synth.random_rows(m, n, seed=r)), device="cuda")
        csr = sq.CsrMetric(rp, ci, vals, halo=1)
        try:
            return sq.scqr3_factor_oblique_csr(Xr, csr, comm=comms[r], stream=streams[r]).status
        except sq.ScqrError as e:
            return str(e)

    out = run_ranks([lambda r=r: call(r) for r in range(P)])
    assert all(isinstance(o, str) for o in out), out
    assert "CSR" in out[P - 1]
    for c in comms:
        c.destroy()


@gpu
def test_loopback_complex_and_gram():
    """The complex path and the kernel-level Gram also sum through the communicator."""
    P = 4
    m, n = 40_000, 24
    Z = synth.randsvd_complex(m, n, 1e9, seed=4)
    ro = oracle.zscqr3(Z)
    comms = sq.Comm.loopback(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    parts = []
    for r in range(P):
        r0, r1 = row_block(m, r, P)
        Zr = torch.from_numpy(np.asfortranarray(Z[r0:r1])).cuda().t().contiguous().t()
        parts.append(Zr)
    torch.cuda.synchronize()
    res = run_ranks([lambda r=r: sq.scqr3_factor_complex(parts[r], comm=comms[r], stream=streams[r], m_global=m)
                     for r in range(P)])
    assert all(x.status == 0 for x in res)
    R0 = res[0].R.cpu().numpy()
    assert all(np.array_equal(x.R.cpu().numpy(), R0) for x in res)
    assert np.max(np.abs(R0 - ro.R)) <= 1e-10 * np.max(np.abs(ro.R))
    Q = np.concatenate([x.Q.cpu().numpy() for x in res], axis=0)
    assert oracle.zorth_F(Q) <= 10 * n * U
    # kernel-level Gram with the communicator: the sum of the shard Grams
    X = synth.random_rows(m, 40, seed=9)
    Xs = [sq.to_colmajor(torch.from_numpy(np.asfortranarray(X[slice(*row_block(m, r, P))])), device="cuda")
          for r in range(P)]
    torch.cuda.synchronize()
    As = run_ranks([lambda r=r: sq.scqr3_gram(Xs[r], comm=comms[r], stream=streams[r]).cpu().numpy()
                    for r in range(P)])
    Ao = oracle.gram(X)
    bound = 2 * (m * U) * (np.abs(X).T @ np.abs(X))
    for A in As:
        assert np.array_equal(A, As[0])
        assert np.all(np.abs(A - Ao) <= bound)
    for c in comms:
        c.destroy()


@gpu
@pytest.mark.parametrize("deterministic", [False, True])
def test_loopback_complex_wide(deterministic):
    """Complex n > 256 across ranks: the three Gram pieces (two block Grams and the cross block)
    sum through one allreduce; R identical on every rank and equal to the oracle's."""
    P = 3
    m, n = 9_000, 272
    Z = synth.randsvd_complex(m, n, 1e10, seed=6)
    ro = oracle.zscqr3(Z)
    comms = sq.Comm.loopback(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    parts = []
    for r in range(P):
        r0, r1 = row_block(m, r, P)
        parts.append(torch.from_numpy(np.asfortranarray(Z[r0:r1])).cuda().t().contiguous().t())
    torch.cuda.synchronize()
    res = run_ranks([lambda r=r: sq.scqr3_factor_complex(parts[r], comm=comms[r], stream=streams[r], m_global=m,
                                                         deterministic=deterministic) for r in range(P)])
    assert all(x.status == 0 for x in res)
    R0 = res[0].R.cpu().numpy()
    assert all(np.array_equal(x.R.cpu().numpy(), R0) for x in res)
    assert np.max(np.abs(R0 - ro.R)) <= 1e-10 * np.max(np.abs(ro.R))
    Q = np.concatenate([x.Q.cpu().numpy() for x in res], axis=0)
    assert oracle.zorth_F(Q) <= 10 * n * U
    for c in comms:
        c.destroy()


@gpu
def test_ghost_plan_single_rank_and_rejection():
    """The ghost-plan CSR mode on one GPU (no communicator: nghost = 0) equals the plain CSR
    call bit for bit; across ranks, a send count that does not match the receiver's recv count
    makes every rank return SCQR3_EINVAL before any exchange."""
    X, B = _inputs("csr_ghost")
    m, n = 20_000, 32
    Xs = np.asfortranarray(X[:m, :n])
    rp, ci, cv = synth.csr_rows(B, 0, m)
    keep = (ci >= 0) & (ci < m)   # drop the couplings out of the first block: an SPD principal block
    rows = np.repeat(np.arange(m), np.diff(rp))[keep]
    nrp = np.zeros(m + 1, dtype=np.int64)
    np.add.at(nrp, rows + 1, 1)
    nrp = np.cumsum(nrp)
    Xd = sq.to_colmajor(torch.from_numpy(Xs), device="cuda")
    a = sq.scqr3_factor_oblique_csr(Xd, sq.CsrMetric(nrp, ci[keep], cv[keep]))
    g = sq.scqr3_factor_oblique_csr(Xd, sq.CsrMetric(nrp, ci[keep], cv[keep],
                                                     ghosts=(0, np.zeros(1), np.zeros(1), np.zeros(0))))
    assert a.status == g.status == 0
    assert np.array_equal(a.R.cpu().numpy(), g.R.cpu().numpy())
    # inconsistent plan over 2 ranks: rank 0 claims one row more than rank 1 expects
    P = 2
    pls = [dict(p) for p in _plans(P)]
    pls[0]["send_counts"] = pls[0]["send_counts"].copy()
    pls[0]["send_counts"][1] += 1
    pls[0]["send_rows"] = np.concatenate([pls[0]["send_rows"], [0]])
    comms = sq.Comm.loopback(P)
    try:
        args = []
        for r in range(P):
            r0, r1 = row_block(M, r, P)
            pl = pls[r]
            csr = sq.CsrMetric(pl["row_ptr"], pl["col_idx"], pl["vals"],
                               ghosts=(pl["nghost"], pl["recv_counts"], pl["send_counts"], pl["send_rows"]))
            Xr = sq.to_colmajor(torch.from_numpy(np.asfortranarray(X[r0:r1])), device="cuda")
            args.append((Xr, csr, dict(comm=comms[r], stream=torch.cuda.Stream())))

        def call(a):
            try:
                return sq.scqr3_factor_oblique_csr(a[0], a[1], **a[2]).status
            except sq.ScqrError as e:
                return str(e)

        out = run_ranks([lambda a=a: call(a) for a in args])
        assert all(isinstance(o, str) for o in out), out
        assert "ghost plan" in out[1] and "rank 1" in out[0], out
    finally:
        for c in comms:
            c.destroy()


@gpu
def test_ghost_plan_with_empty_rank():
    """A ghost-plan CSR factorisation over 3 loopback ranks, the middle one owning no rows: its
    plan is empty, the others exchange with each other only; R matches the oracle's 2-part
    emulation (an empty shard adds zeros) and every rank returns the same R."""
    X, B = _inputs("csr_ghost")
    h = M // 2
    bounds = [(0, h), (h, h), (h, M)]
    # plans for the 2-rank split, with an empty rank spliced in between
    p2 = _plans(2)
    empty = dict(row_ptr=np.zeros(1, dtype=np.int64), col_idx=np.zeros(0, dtype=np.int32), vals=np.zeros(0),
                 nghost=0, recv_counts=np.zeros(3, dtype=np.int64), send_counts=np.zeros(3, dtype=np.int64),
                 send_rows=np.zeros(0, dtype=np.int64))
    def widen(pl):
        q = dict(pl)
        q["recv_counts"] = np.array([pl["recv_counts"][0], 0, pl["recv_counts"][1]], dtype=np.int64)
        q["send_counts"] = np.array([pl["send_counts"][0], 0, pl["send_counts"][1]], dtype=np.int64)
        return q
    plans = [widen(p2[0]), empty, widen(p2[1])]
    comms = sq.Comm.loopback(3)
    streams = [torch.cuda.Stream() for _ in range(3)]
    n = X.shape[1]
    args = []
    for r, (r0, r1) in enumerate(bounds):
        pl = plans[r]
        csr = sq.CsrMetric(pl["row_ptr"], pl["col_idx"], pl["vals"],
                           ghosts=(pl["nghost"], pl["recv_counts"], pl["send_counts"], pl["send_rows"]))
        Xr = sq.to_colmajor(torch.from_numpy(np.asfortranarray(X[r0:r1])), device="cuda") if r1 > r0 else \
            sq.colmajor_empty(0, n)
        args.append((Xr, csr, dict(comm=comms[r], stream=streams[r])))
    try:
        res = run_ranks([lambda a=a: sq.scqr3_factor_oblique_csr(a[0], a[1], **a[2]) for a in args])
    finally:
        for c in comms:
            c.destroy()
    assert all(x.status == 0 for x in res)
    R0 = res[0].R.cpu().numpy()
    assert all(np.array_equal(x.R.cpu().numpy(), R0) for x in res)
    ro = _oracle("csr_ghost", 2)
    assert np.max(np.abs(R0 - ro.R)) <= 1e-10 * np.max(np.abs(ro.R))


@gpu
def test_loopback_host_batch():
    """scqr3_factor_host_batch with a loopback communicator: every rank streams the same number of
    matrices (its row block of each); per matrix, R is identical on every rank and equals the
    per-call multi-rank result."""
    P, m, n, count = 2, 40_000, 48, 3
    Xs = [synth.randsvd(m, n, 10.0 ** (4 + 3 * i), seed=30 + i) for i in range(count)]
    parts = [row_block(m, r, P) for r in range(P)]

    def pin(A=None, shape=None):
        T = torch.empty(shape[::-1], dtype=torch.float64, pin_memory=True)
        if A is not None:
            T.copy_(torch.from_numpy(np.ascontiguousarray(A.T)))
        return T.t()

    comms = sq.Comm.loopback(P)
    streams = [torch.cuda.Stream() for _ in range(P)]
    try:
        Xh = [[pin(X[a:b], (b - a, n)) for X in Xs] for a, b in parts]
        Qh = [[pin(shape=(b - a, n)) for _ in Xs] for a, b in parts]
        Rh = [[pin(shape=(n, n)) for _ in Xs] for _ in parts]
        st = run_ranks([lambda r=r: sq.scqr3_factor_host_batch(Xh[r], Qh[r], Rh[r], comm=comms[r], m_global=m,
                                                               stream=streams[r]) for r in range(P)])
        assert st == [[0] * count] * P
        for i in range(count):
            assert np.array_equal(Rh[0][i].numpy(), Rh[1][i].numpy())
            one = run_ranks([lambda r=r: sq.scqr3_factor_host(Xh[r][i], comm=comms[r], m_global=m, stream=streams[r])
                             for r in range(P)])
            assert np.array_equal(one[0].R.numpy(), Rh[0][i].numpy())
            assert all(np.array_equal(one[r].Q.numpy(), Qh[r][i].numpy()) for r in range(P))
    finally:
        for c in comms:
            c.destroy()
