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


def _device_view(ptr: int, count: int, device) -> torch.Tensor:
    """A float64 tensor over library-owned device memory (no copy, no ownership)."""
    class _V:
        def __init__(self):
            self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False),
                                             "version": 3, "strides": None}
    return torch.as_tensor(_V(), device=device)


class FusedExchangeSpMV:
    """Row-sharded iterated merge-CSR with the exchange fused into the multiply (SURVEY §8e,
    stretch): every rank owns two exchange buffers of the full x (ping-pong) that all ranks map
    through CUDA IPC; a step multiplies the local rows and the kernel epilogue stores each finished
    row straight into the next-x buffer of every rank (own rows locally, the others over NVLink /
    NVSwitch peer stores) -- no separate all-gather pass over y.  A rank barrier ends the step.

    `fmt` is the rank's CRS-family shard format (rows [lo, hi), global columns); `barrier` is a
    callable (default torch.distributed.barrier on `group`)."""

    def __init__(self, cuts: Sequence[int], rank: int, fmt, n: int, group=None, barrier=None):
        import ctypes as C
        import torch.distributed as dist
        from . import capi
        from .engine import _check
        self.C, self.capi, self._check = C, capi, _check
        L = capi.load()
        self.cuts = list(cuts)
        self.rank, self.world = rank, len(cuts) - 1
        self.lo, self.hi = self.cuts[rank], self.cuts[rank + 1]
        self.fmt, self.n = fmt, n
        # the shards must tile a square matrix: every rank's rows land in every peer's n-long
        # buffer at their row offset (checked again by the library per multiply)
        shape_err = None
        if self.cuts[0] != 0 or self.cuts[-1] != n or any(a > b for a, b in zip(self.cuts, self.cuts[1:])):
            shape_err = f"row cuts {self.cuts[0]}..{self.cuts[-1]} do not tile the n = {n} exchange buffers"
        elif fmt.m != self.hi - self.lo or fmt.n != n:
            shape_err = f"shard format is {fmt.m} x {fmt.n}, expected {self.hi - self.lo} x {n}"
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.group = group
        self.barrier = barrier or (lambda: dist.barrier(group))
        # Over NCCL the end-of-step rendezvous is a stream-ordered 1-element all-reduce: a rank's
        # next multiply cannot start before every rank's scatter kernels completed (their peer
        # stores are performed at kernel completion), and the host never waits.
        self._stream_barrier = barrier is None and dist.get_backend(group) == "nccl"
        self._token = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.own, handles, err = [], [], shape_err
        try:
            if err is not None:
                raise ValueError(err)
            for _ in range(2):
                p, h = C.c_void_p(), (C.c_ubyte * 64)()
                _check(L.spmvlab_cuda_exchange_alloc(8 * max(n, 1), C.byref(p), h))
                self.own.append(p.value)
                handles.append(bytes(h))
        except Exception as e:  # agree on failure collectively instead of leaving peers waiting
            err = repr(e)
        every = [None] * self.world
        dist.all_gather_object(every, (err, handles), group)
        self.opened = []
        self.ptr = [[0] * self.world for _ in range(2)]  # ptr[buffer][rank], mapped into this process
        if err is None and all(e is None for e, _ in every):
            try:
                for q in range(self.world):
                    for b in range(2):
                        if q == rank:
                            self.ptr[b][q] = self.own[b]
                            continue
                        p = C.c_void_p()
                        _check(L.spmvlab_cuda_exchange_open((C.c_ubyte * 64).from_buffer_copy(every[q][1][b]),
                                                            C.byref(p)))
                        self.ptr[b][q] = p.value
                        self.opened.append(p.value)
            except Exception as e:
                err = repr(e)
        else:
            err = err or next(e for e, _ in every if e is not None)
        status = [None] * self.world
        dist.all_gather_object(status, err, group)
        failed = [s for s in status if s is not None]
        if failed:
            for p in self.opened:
                L.spmvlab_cuda_exchange_close(p, 1)
            self.barrier()
            for p in self.own:
                L.spmvlab_cuda_exchange_close(p, 0)
            self.opened, self.own = [], []
            raise RuntimeError(f"fused exchange unavailable: {failed[0]}")
        self.cur = 0

    def x(self) -> torch.Tensor:
        """This rank's copy of the current iterate (a view of the exchange buffer)."""
        return _device_view(self.ptr[self.cur][self.rank], self.n, self.device)

    def load(self, x0: torch.Tensor) -> None:
        self.x().copy_(x0)
        torch.cuda.synchronize()
        self.barrier()

    def step(self, stream=None) -> None:
        C = self.C
        nxt = 1 - self.cur
        peers = [self.ptr[nxt][q] for q in range(self.world) if q != self.rank]
        dest = (C.c_void_p * max(len(peers), 1))(*peers)
        st = stream or torch.cuda.current_stream()
        y_local = self.ptr[nxt][self.rank] + 8 * self.lo  # own rows go straight into the own next x
        self._check(self.capi.load().spmvlab_cuda_run_spmv_scatter(
            self.fmt.handle, self.ptr[self.cur][self.rank], self.n, y_local, self.hi - self.lo, dest, len(peers),
            self.n, self.lo, st.cuda_stream))
        if self._stream_barrier:
            import torch.distributed as dist
            with torch.cuda.stream(st):
                dist.all_reduce(self._token, group=self.group)
        else:
            st.synchronize()
            self.barrier()  # every rank's rows have landed in every next buffer
        self.cur = nxt

    def iterate(self, x0: torch.Tensor, iters: int) -> torch.Tensor:
        self.load(x0)
        for _ in range(iters):
            self.step()
        return self.x().clone()

    def close(self) -> None:
        """Collective: unmaps the peers' buffers, then (after every rank did) frees its own."""
        L = self.capi.load()
        torch.cuda.synchronize()
        self.barrier()
        for p in self.opened:
            L.spmvlab_cuda_exchange_close(p, 1)
        self.barrier()
        for p in self.own:
            L.spmvlab_cuda_exchange_close(p, 0)
        self.opened, self.own = [], []
