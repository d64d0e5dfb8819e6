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
