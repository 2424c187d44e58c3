"""Row-sharded (iterated) SpMV across ranks: SURVEY.md §8(e).

A is split into contiguous row ranges balanced by nonzeros with the reference's own greedy cut,
partition_rows_by_nnz with beta = 1 (inc/block_size.hpp:73-102, inc/triplet.hpp:82-87).  Each rank
keeps its rows (global column indices) and a full replica of x; one step is the local multiply
y_r = A_r x followed by the variable-count all-gather of the y_r slices into every rank's copy of
y (x of the next iteration).  The shard row counts differ by ~89x on power-law matrices, so the
all-gather is a group of per-rank broadcasts (an all-gatherv), not a padded all_gather.

The local multiply is a callable: on GPUs it is the CUDA merge-CSR engine over NCCL
(bench.py); the gloo tests plug in a CPU multiply to check the sharding and exchange logic.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np
import torch


def row_prefix(m: int, rows) -> np.ndarray:
    """Exclusive prefix of per-row counts, length m + 1 (inc/triplet.hpp:82-87)."""
    rows = rows.cpu().numpy() if isinstance(rows, torch.Tensor) else np.asarray(rows)
    counts = np.bincount(rows.astype(np.int64), minlength=m)
    prefix = np.zeros(m + 1, dtype=np.uint64)
    prefix[1:] = np.cumsum(counts)
    return prefix


def shard_bounds(prefix: np.ndarray, world: int) -> list[int]:
    """Row cuts [0, c1, ..., m] of a nonzero-balanced world-way split (beta = 1)."""
    from .engine import partition_rows_by_nnz
    if int(prefix[-1]) > 0xFFFFFFFF:
        raise ValueError("nnz exceeds the 32-bit index type")
    return [int(b) for b in partition_rows_by_nnz(prefix.astype(np.uint32), world, 0)]


def shard_rows(rows, cols, vals, lo: int, hi: int):
    """Entries of rows [lo, hi) with row indices made local (columns stay global)."""
    if isinstance(rows, torch.Tensor):
        sel = (rows >= lo) & (rows < hi)
        return (rows[sel] - lo).to(torch.int32).contiguous(), cols[sel].contiguous(), vals[sel].contiguous()
    rows = np.asarray(rows)
    sel = (rows >= lo) & (rows < hi)
    return (rows[sel] - lo).astype(np.uint32), np.asarray(cols)[sel], np.asarray(vals)[sel]


def allgatherv_(y_full: torch.Tensor, cuts: Sequence[int], group=None) -> torch.Tensor:
    """In place: rank q's slice y_full[cuts[q]:cuts[q+1]] is broadcast to every rank."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    works = []
    for q in range(world):
        lo, hi = cuts[q], cuts[q + 1]
        if hi > lo:
            works.append(dist.broadcast(y_full[lo:hi], src=q, group=group, async_op=True))
    for w in works:
        w.wait()
    return y_full


class ShardedSpMV:
    """One rank's share of y = A x with the all-gatherv exchange."""

    def __init__(self, cuts: Sequence[int], rank: int, local_multiply: Callable, group=None):
        self.cuts = list(cuts)
        self.rank = rank
        self.lo, self.hi = self.cuts[rank], self.cuts[rank + 1]
        self.local_multiply = local_multiply  # (x_full, y_local_view) -> None
        self.group = group

    def step(self, x: torch.Tensor, y_full: torch.Tensor) -> torch.Tensor:
        self.local_multiply(x, y_full[self.lo:self.hi])
        return allgatherv_(y_full, self.cuts, self.group)

    def iterate(self, x0: torch.Tensor, iters: int) -> torch.Tensor:
        """x_{k+1} = A x_k, iters times; returns x_iters on every rank."""
        x = x0.clone()
        y = torch.empty_like(x0)
        for _ in range(iters):
            self.step(x, y)
            x, y = y, x
        return x
