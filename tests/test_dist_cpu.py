"""World-size-2 gloo tests of the row-sharded iterated SpMV host logic on CPU.

The local multiply is the C oracle's sequential CRS (test infrastructure), so every row is summed
in the reference order and the sharded result must be BITWISE equal to the single-process oracle
loop at iterations 1, 2 and 5 (column-normalised R-MAT, non-negative x0, as cfg5)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix():
    from paper_2502_19284_b200 import gen
    return gen.rmat_host(10, 8, seed=11, normalize_columns=True)


def _worker(rank, world, port, iters, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_2502_19284_b200 import dist as sd
        orc = Oracle()
        m, n, r, c, v = _matrix()
        cuts = sd.shard_bounds(sd.row_prefix(m, r), world)
        lr, lc, lv = sd.shard_rows(r, c, v, cuts[rank], cuts[rank + 1])
        local = orc.build(0, cuts[rank + 1] - cuts[rank], n, lr, lc, lv)

        def multiply(x_full, y_local):
            y_local.copy_(torch.from_numpy(orc.spmv(local, 0, x_full.numpy())))

        sh = sd.ShardedSpMV(cuts, rank, multiply)
        x0 = torch.from_numpy(np.random.default_rng(5).uniform(0.0, 1.0, n))
        outs = [sh.iterate(x0, k).numpy().copy() for k in iters]
        out_q.put((rank, cuts, outs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_iterated_spmv_matches_oracle(world, oracle):
    iters = (1, 2, 5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m, n, r, c, v = _matrix()
    full = oracle.build(0, m, n, r, c, v)
    x = np.random.default_rng(5).uniform(0.0, 1.0, n)
    want = {}
    xk = x.copy()
    for k in range(1, max(iters) + 1):
        xk = oracle.spmv(full, 0, xk)
        want[k] = xk.copy()
    for rank, cuts, outs in results:
        assert cuts[0] == 0 and cuts[-1] == m and len(cuts) == world + 1
        for k, got in zip(iters, outs):
            np.testing.assert_array_equal(got, want[k], err_msg=f"rank {rank} iteration {k}")


def test_shard_bounds_match_reference_partition(oracle):
    """The cuts are partition_rows_by_nnz(prefix, p, beta=1) (inc/block_size.hpp:73-102)."""
    from paper_2502_19284_b200 import dist as sd
    m, n, r, c, v = _matrix()
    prefix = sd.row_prefix(m, r)
    for p in (1, 2, 3, 4, 8):
        assert sd.shard_bounds(prefix, p) == oracle.partition_rows_by_nnz(prefix.astype(np.uint32), p, 0).tolist()
