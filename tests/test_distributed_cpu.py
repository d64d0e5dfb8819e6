"""World-size-2 gloo tests (CPU) of the multi-rank decomposition that libscqr3 runs over NCCL:
row-block partition, Gram allreduce (sum of per-rank Grams), replicated Cholesky on identical
bits, local TRSM, oblique one-row halo exchange, and max-over-ranks timing.  The arithmetic of
each rank is the oracle's; only the exchange pattern is under test here."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1809_11085_b200 import dist as pdist  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import oracle
    import synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n = 3001, 12
        X = synth.randsvd(m, n, 1e12, seed=5)
        d, e = synth.tridiag_b(m, seed=5)
        r0, r1 = pdist.row_block(m, rank, world)
        Xl = np.asfortranarray(X[r0:r1])
        res = {}
        # ---- standard inner product: Gram allreduce + replicated Cholesky + local TRSM
        Q = Xl.copy(order="F")
        R = np.eye(n)
        for k in range(3):
            A = torch.from_numpy(oracle.gram(Q))
            dist.all_reduce(A)                                   # the one exchange per pass
            A = A.numpy()
            s = oracle.shift(m, n, oracle.power_lmax(A) * 1.01) if k == 0 else 0.0   # global m
            Rt = oracle.cholesky(A, s)
            Q = oracle.trsm_rows(Q, Rt)
            R = oracle.trmul(Rt, R)
        res["R"] = R
        res["Qrows"] = (r0, Q)
        # ---- oblique: halo rows from the neighbours give the same rows of Y = B X
        up, down = pdist.neighbours(rank, world)
        first, last = torch.from_numpy(Xl[0].copy()), torch.from_numpy(Xl[-1].copy())
        halo_prev, halo_next = torch.zeros(n, dtype=torch.float64), torch.zeros(n, dtype=torch.float64)
        ops = []
        if up is not None:
            ops += [dist.P2POp(dist.isend, first, up), dist.P2POp(dist.irecv, halo_prev, up)]
        if down is not None:
            ops += [dist.P2POp(dist.isend, last, down), dist.P2POp(dist.irecv, halo_next, down)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        Y = d[r0:r1, None] * Xl
        Y[1:] += e[r0:r1 - 1, None] * Xl[:-1]
        Y[:-1] += e[r0:r1 - 1, None] * Xl[1:]
        if up is not None:
            Y[0] += e[r0 - 1] * halo_prev.numpy()
        if down is not None:
            Y[-1] += e[r1 - 1] * halo_next.numpy()
        res["Yrows"] = (r0, Y)
        # ---- CSR metric: libscqr3's h-row halo protocol -- first h rows to
        # the previous rank, last h rows to the next; column indices relative to the rank's
        # first row, [-h, 0) -> previous rank's rows, [m_loc, m_loc + h) -> next rank's rows
        nx, ny = 30, 40
        mc = nx * ny
        Bc = synth.laplacian2d(nx, ny, seed=1, wmax=10.0)
        Xc = synth.randsvd(mc, n, 1e6, seed=6)
        c0, c1 = pdist.row_block(mc, rank, world)
        rp, ci, cv = synth.csr_rows(Bc, c0, c1)
        h = nx                                                  # grid width = band half-width
        Xcl = Xc[c0:c1]
        hp, hn = torch.zeros((h, n), dtype=torch.float64), torch.zeros((h, n), dtype=torch.float64)
        ops = []
        if up is not None:
            ops += [dist.P2POp(dist.isend, torch.from_numpy(Xcl[:h].copy()), up), dist.P2POp(dist.irecv, hp, up)]
        if down is not None:
            ops += [dist.P2POp(dist.isend, torch.from_numpy(Xcl[-h:].copy()), down),
                    dist.P2POp(dist.irecv, hn, down)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        ext = np.vstack([hp.numpy(), Xcl, hn.numpy()])          # rows -h .. m_loc + h - 1
        assert ci.min() >= -h and ci.max() < (c1 - c0) + h
        Yc = np.zeros_like(Xcl)
        for i in range(c1 - c0):
            for z in range(rp[i], rp[i + 1]):
                Yc[i] += cv[z] * ext[ci[z] + h]
        G = torch.from_numpy(np.asfortranarray(Xcl.T @ Yc))
        dist.all_reduce(G)
        res["Gcsr"] = G.numpy()
        res["tmax"] = pdist.max_over_ranks(1.0 + rank)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_partition_covers_rows_once():
    for m, w in [(10, 3), (1, 2), (10_000_000, 8), (7, 8)]:
        blocks = [pdist.row_block(m, r, w) for r in range(w)]
        assert blocks[0][0] == 0 and blocks[-1][1] == m
        assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))
        sizes = [b - a for a, b in blocks]
        assert max(sizes) - min(sizes) <= 1


def test_two_rank_gloo_decomposition_matches_single_process():
    import oracle
    import synth

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # replicated Cholesky on identical allreduced Grams -> identical R bits on every rank
    assert np.array_equal(out[0]["R"], out[1]["R"])
    m, n = 3001, 12
    X = synth.randsvd(m, n, 1e12, seed=5)
    ref = oracle.scqr3(X, max_passes=3, nparts=2)        # the oracle's own 2-rank emulation
    assert np.max(np.abs(out[0]["R"] - ref.R)) <= 1e-10 * np.max(np.abs(ref.R))
    Q = np.zeros((m, n))
    for rank in range(world):
        r0, Ql = out[rank]["Qrows"]
        Q[r0:r0 + Ql.shape[0]] = Ql
    assert oracle.orth_F(Q) <= 10 * n * 2.0 ** -53
    # halo exchange reproduces the global B X
    d, e = synth.tridiag_b(m, seed=5)
    B = np.diag(d) + np.diag(e[:-1], 1) + np.diag(e[:-1], -1)
    Yg = B @ X
    for rank in range(world):
        r0, Yl = out[rank]["Yrows"]
        assert np.allclose(Yl, Yg[r0:r0 + Yl.shape[0]], rtol=1e-14, atol=1e-12)
    assert out[0]["tmax"] == out[1]["tmax"] == 2.0
    # CSR halo protocol: the allreduced per-rank X^T (B X) equals the global Gram
    Bc = synth.laplacian2d(30, 40, seed=1, wmax=10.0)
    Xc = synth.randsvd(1200, n, 1e6, seed=6)
    Ac, _ = oracle.gram_oblique_csr(Xc, Bc)
    G = out[0]["Gcsr"]
    assert np.array_equal(G, out[1]["Gcsr"])
    assert np.max(np.abs((G + G.T) / 2 - Ac)) <= 1e-12 * np.max(np.abs(Ac))


def _gen_worker(rank, world, port, q):
    import synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        synth.CHUNK_ROWS = 1 << 12           # several chunks, some split between ranks
        m, n = 20_000, 6
        r0, r1 = pdist.row_block(m, rank, world)
        X = synth.randsvd_torch_rows(m, n, 1e8, r0, r1, seed=3, device="cpu", allreduce=dist.all_reduce)
        q.put((rank, (r0, X.numpy().copy())))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_row_sharded_generator_matches_one_rank():
    """bench.py's multi-GPU input: each rank generates only its rows (per-chunk seeded Gaussian
    chunks, Householder TSQR with the chunk R factors summed over ranks); the stitched X is
    bitwise the one-rank X, with the requested spectrum."""
    import synth

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gen_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    synth.CHUNK_ROWS = 1 << 12
    try:
        ref = synth.randsvd_torch(20_000, 6, 1e8, seed=3, device="cpu").numpy()
    finally:
        synth.CHUNK_ROWS = 1 << 20
    X = np.concatenate([out[r][1] for r in range(world)], axis=0)
    assert np.array_equal(X, ref)
    s = np.linalg.svd(X, compute_uv=False)
    assert abs(s[0] - 1.0) < 1e-12 and abs(s[0] / s[-1] / 1e8 - 1.0) < 1e-6


def test_csr_ghost_plan_reproduces_global_spmv():
    """dist.csr_ghost_plan (host bookkeeping for the SCQR3_CSR_GHOSTS exchange): for a Laplacian
    whose rows and columns are randomly permuted (no band), every rank's local CSR applied to
    [its rows; the ghost rows its peers send, in plan order] equals the rows of the global B @ X,
    and rank r's send counts match every peer's receive counts (the collective check the library
    makes).  Pure numpy, P = 1..5 (including a rank with no rows)."""
    import synth
    from paper_1809_11085_b200.dist import csr_ghost_plan, row_block

    rp, ci, cv = synth.laplacian2d(30, 20, seed=0, wmax=10.0)
    m = len(rp) - 1
    perm = np.random.default_rng(1).permutation(m)
    inv = np.empty(m, dtype=np.int64)
    inv[perm] = np.arange(m)
    cnt = np.diff(rp)
    nrp = np.concatenate([[0], np.cumsum(cnt[perm])])
    idx = np.concatenate([np.arange(rp[o], rp[o + 1]) for o in perm])
    nci, ncv = inv[ci[idx]], cv[idx]
    X = np.random.default_rng(2).standard_normal((m, 3))
    Y = np.zeros_like(X)
    for i in range(m):
        for z in range(nrp[i], nrp[i + 1]):
            Y[i] += ncv[z] * X[nci[z]]
    for P in (1, 2, 3, 5):
        plans = csr_ghost_plan(nrp, nci, ncv, m, P)
        for r in range(P):
            for p in range(P):
                assert plans[r]["send_counts"][p] == plans[p]["recv_counts"][r]
            assert plans[r]["recv_counts"][r] == 0 and plans[r]["send_counts"][r] == 0
        for r in range(P):
            r0, r1 = row_block(m, r, P)
            pl = plans[r]
            ghost = []
            for p in range(P):   # what rank p packs for rank r, in its send order
                p0, _ = row_block(m, p, P)
                off = int(np.sum(plans[p]["send_counts"][:r]))
                rows = plans[p]["send_rows"][off:off + plans[p]["send_counts"][r]]
                ghost.append(X[p0 + rows])
            G = np.concatenate([X[r0:r1]] + ghost) if ghost else X[r0:r1]
            assert G.shape[0] == (r1 - r0) + pl["nghost"]
            Yr = np.zeros((r1 - r0, 3))
            for i in range(r1 - r0):
                for z in range(pl["row_ptr"][i], pl["row_ptr"][i + 1]):
                    Yr[i] += pl["vals"][z] * G[pl["col_idx"][z]]
            assert np.array_equal(Yr, Y[r0:r1])
    # a rank with no rows: row_block(m=5, P=8) gives empty blocks
    plans = csr_ghost_plan(np.arange(6, dtype=np.int64), np.arange(5), np.ones(5), 5, 8)
    assert sum(p["nghost"] for p in plans) == 0
