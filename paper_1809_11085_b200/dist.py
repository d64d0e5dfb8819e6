"""Multi-GPU plumbing shared by bench.py and the tests: row-block partition and rank helpers.

The method's only exchange is the sum of the per-rank Grams ("reduction operator is
addition"), done inside libscqr3 by one NCCL allreduce per pass; the oblique variant also swaps
one boundary row with each neighbour.  This module holds no arithmetic of the method.
"""
from __future__ import annotations


def row_block(m: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous rows [r0, r1) of rank `rank` (sizes differ by at most one)."""
    if not (0 <= rank < world):
        raise ValueError("bad rank")
    return m * rank // world, m * (rank + 1) // world


def neighbours(rank: int, world: int) -> tuple[int | None, int | None]:
    """Ranks holding the rows just above / below this rank's block (oblique halo)."""
    return (rank - 1 if rank > 0 else None), (rank + 1 if rank + 1 < world else None)


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Max of a per-rank time over all ranks (benchmarks report the slowest rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


_POOL = None


def run_ranks(fns):
    """Run fns[r]() for every rank r concurrently, one host thread per rank (the loopback
    communicator's ranks, scqr3_comm_init_loopback), and return their results in rank order.
    The threads are reused across calls (each thread keeps the library's per-thread state).
    An exception in any rank is re-raised after all ranks have returned."""
    import concurrent.futures as cf

    global _POOL
    if _POOL is None or _POOL._max_workers < len(fns):
        _POOL = cf.ThreadPoolExecutor(max_workers=max(16, len(fns)), thread_name_prefix="scqr3-rank")
    futs = [_POOL.submit(f) for f in fns]
    out, err = [], None
    for f in futs:
        try:
            out.append(f.result())
        except BaseException as e:  # noqa: BLE001 -- re-raised below after every rank returned
            out.append(None)
            err = err or e
    if err is not None:
        raise err
    return out


def csr_ghost_plan(row_ptr, col_idx, vals, m: int, world: int):
    """Split a global CSR matrix (numpy: row_ptr int64[m+1], col_idx global indices, vals) into
    the row blocks of `row_block` and build each rank's ghost-row plan (include/scqr3.h,
    SCQR3_CSR_GHOSTS) -- the distributed sparse matrix-vector product layout, for any sparsity
    pattern.  Returns, per rank r, a dict with the local CSR (`row_ptr`, `col_idx` int32 with
    ghost rows at m_r + slot, `vals`) and the plan (`nghost`, `recv_counts`, `send_counts`,
    `send_rows`): ghost slots are ordered by owning rank, then by global row; rank p's send list
    to r is r's ghost rows from p in the same order, as p-local row indices.  Index bookkeeping
    only -- no arithmetic of the method."""
    import numpy as np

    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col_idx = np.asarray(col_idx, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    bounds = np.array([row_block(m, r, world)[0] for r in range(world)] + [m], dtype=np.int64)
    need = []      # need[r][p]: sorted global rows rank r reads from rank p
    local = []
    for r in range(world):
        r0, r1 = int(bounds[r]), int(bounds[r + 1])
        z0, z1 = int(row_ptr[r0]), int(row_ptr[r1])
        cols = col_idx[z0:z1]
        owner = np.searchsorted(bounds, cols, side="right") - 1
        remote = owner != r
        need_r = [np.unique(cols[remote & (owner == p)]) for p in range(world)]
        need.append(need_r)
        slot_base = np.cumsum([0] + [len(x) for x in need_r])
        lc = np.empty(len(cols), dtype=np.int64)
        lc[~remote] = cols[~remote] - r0
        for p in range(world):
            sel = remote & (owner == p)
            if sel.any():
                lc[sel] = (r1 - r0) + slot_base[p] + np.searchsorted(need_r[p], cols[sel])
        local.append(dict(row_ptr=row_ptr[r0:r1 + 1] - z0, col_idx=lc.astype(np.int32), vals=vals[z0:z1],
                          nghost=int(slot_base[-1]), recv_counts=np.array([len(x) for x in need_r], dtype=np.int64)))
    for p in range(world):
        p0 = int(bounds[p])
        lists = [need[r][p] - p0 for r in range(world)]
        local[p]["send_counts"] = np.array([len(x) for x in lists], dtype=np.int64)
        local[p]["send_rows"] = (np.concatenate(lists) if lists else np.zeros(0)).astype(np.int64)
    return local
