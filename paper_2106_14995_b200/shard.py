"""Multi-GPU sharding of a batch: one process per GPU (torch.distributed),
contiguous even partitions in input order exactly like the reference's
static worker partition (batch.hpp:61-70: base = n / workers, the first
n % workers partitions get one extra problem).  Problems are independent, so
the data path has no collective; results are gathered only if asked.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple

import numpy as np

from .tron import BatchResult, ProblemBatch

FIELDS = ("x_star", "f_star", "pg_norm", "status", "iterations", "cg_iterations", "f_evals")


def partition(count: int, parts: int) -> List[Tuple[int, int]]:
    """[lo, hi) of each partition (batch.hpp:61-70)."""
    if parts < 1:
        raise ValueError("solve_batch: workers must be >= 1")
    base, rem = divmod(count, parts)
    out, lo = [], 0
    for k in range(parts):
        hi = lo + base + (1 if k < rem else 0)
        out.append((lo, hi))
        lo = hi
    return out


def shard(batch: ProblemBatch, rank: int, world: int) -> Tuple[ProblemBatch, int, int]:
    lo, hi = partition(batch.count, world)[rank]
    sl = slice(lo, hi)
    prm = None if batch.params is None else batch.params[sl]
    x0 = None if batch.x0 is None else batch.x0[sl]
    return ProblemBatch(batch.family, batch.dim, batch.lower[sl], batch.upper[sl], prm, x0), lo, hi


def solve_sharded(batch: ProblemBatch, rank: int, world: int, solve: Callable[[ProblemBatch], object],
                  gather: bool = True, group=None) -> Optional[dict]:
    """Solve this rank's shard with `solve` (e.g. Solver((local_rank,)).solve_batch)
    and, if `gather`, all-gather every SolveReport field into full-size host
    arrays on every rank (torch.distributed, any backend)."""
    import torch
    import torch.distributed as dist

    local, lo, hi = shard(batch, rank, world)
    res = solve(local)
    if not gather:
        return None
    parts = partition(batch.count, world)
    maxlen = max(h - l for l, h in parts)
    out = {}
    for k in FIELDS:
        a = getattr(res, k)
        a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
        pad = np.zeros((maxlen,) + a.shape[1:], dtype=a.dtype)
        pad[: a.shape[0]] = a
        t = torch.from_numpy(pad)
        bufs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(bufs, t, group=group)
        out[k] = np.concatenate([bufs[r].numpy()[: h - l] for r, (l, h) in enumerate(parts)], axis=0)
    return out
