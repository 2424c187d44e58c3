"""The fused multi-GPU exchange (dist.FusedExchangeSpMV: the merge kernel's epilogue stores every
finished row into every rank's next-x buffer through CUDA IPC) with 2 ranks in 2 processes.

Only one GPU is available to this build, so both ranks share cuda:0: the IPC mappings, the peer
stores, the ping-pong buffers and the barrier protocol are exercised for real, while the
kernels never wait on each other (ranks synchronise on the host through gloo).  The iterates
must match the CPU oracle loop (column-normalised R-MAT, x0 > 0: relative 1e-12 per iteration)
and be identical on both ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ITERS = (1, 2, 7)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix():
    from paper_2502_19284_b200 import gen
    return gen.rmat_host(13, 8, seed=17, normalize_columns=True)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2502_19284_b200 as sp
        from paper_2502_19284_b200 import dist as sd
        m, n, r, c, v = _matrix()
        cuts = sd.shard_bounds(sd.row_prefix(m, r), world)
        lr, lc, lv = sd.shard_rows(r, c, v, cuts[rank], cuts[rank + 1])
        fmt = sp.build_format(sp.Algorithm.Merge, sp.TripletMatrix.from_host(cuts[rank + 1] - cuts[rank], n, lr, lc,
                                                                            lv), 1)
        ex = sd.FusedExchangeSpMV(cuts, rank, fmt, n)
        x0 = torch.from_numpy(np.random.default_rng(6).uniform(0.1, 1.0, n)).cuda()
        outs = [ex.iterate(x0, k).cpu().numpy() for k in ITERS]
        ex.close()
        q.put((rank, cuts, outs))
    except Exception as e:  # surface worker failures in the test
        q.put((rank, None, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("panels", [None, 3])
def test_fused_exchange_two_ranks_match_oracle(cuda, oracle, monkeypatch, panels):
    """panels=3: the column-panelled merge engine (only the last panel scatters; rows empty in it
    must still reach the peers)."""
    if panels:
        monkeypatch.setenv("SPMVLAB_MERGE_PANELS", str(panels))  # inherited by the spawned ranks
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, cuts, outs in res:
        assert cuts is not None, f"rank {rank} failed: {outs}"
    m, n, r, c, v = _matrix()
    full = oracle.build(0, m, n, r, c, v)
    x = np.random.default_rng(6).uniform(0.1, 1.0, n)
    want = {}
    for k in range(1, max(ITERS) + 1):
        x = oracle.spmv(full, 0, x)
        want[k] = x.copy()
    by_rank = {rank: outs for rank, _, outs in res}
    for i, k in enumerate(ITERS):
        a, b = by_rank[0][i], by_rank[1][i]
        np.testing.assert_array_equal(a, b)  # every rank holds the same full iterate
        np.testing.assert_allclose(a, want[k], rtol=1e-12 * k, atol=0)
    assert all(p.exitcode == 0 for p in procs)


@pytest.mark.parametrize("panels", [None, 2, 4])
def test_scatter_single_rank_equals_run_spmv(cuda, monkeypatch, panels):
    """World 1: the scatter multiply with no peers is the plain merge multiply (bitwise), and a
    destination list copies every row (including rows finished by the carry fix-up), also with
    column panels."""
    sp = cuda
    import ctypes as C
    from paper_2502_19284_b200 import capi, gen
    from paper_2502_19284_b200.engine import _check
    m, n, r, c, v = gen.rmat_host(12, 16, seed=2)
    if panels:
        monkeypatch.setenv("SPMVLAB_MERGE_PANELS", str(panels))
    f = sp.build_format(2, sp.TripletMatrix.from_host(m, n, r, c, v), 1)
    if panels:
        monkeypatch.delenv("SPMVLAB_MERGE_PANELS")
        assert f.info["merge_panels"] == panels
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y_ref = sp.run_spmv(2, f, x)
    y = torch.empty(m, dtype=torch.float64, device="cuda")
    d1 = torch.full((m + 5,), -1.0, dtype=torch.float64, device="cuda")
    dest = (C.c_void_p * 1)(d1.data_ptr())
    _check(capi.load().spmvlab_cuda_run_spmv_scatter(f.handle, x.data_ptr(), n, y.data_ptr(), m, dest, 1, m + 5,
                                                     5, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    if panels:  # panel 0 runs last with destinations: the same sums in another order
        from parity import assert_y_close
        bound = sp.run_spmv(2, sp.build_format(2, sp.TripletMatrix.from_host(m, n, r, c, np.abs(v)), 1), x.abs())
        assert_y_close(y.cpu().numpy(), y_ref.cpu().numpy(), bound.cpu().numpy(), what=f"panels={panels}")
    else:
        assert torch.equal(y, y_ref)
    assert torch.equal(d1[5:], y) and bool((d1[:5] == -1.0).all())
    # a destination too short for row_offset + m is rejected before anything is written
    rc = capi.load().spmvlab_cuda_run_spmv_scatter(f.handle, x.data_ptr(), n, y.data_ptr(), m, dest, 1, m + 4, 5,
                                                   torch.cuda.current_stream().cuda_stream)
    assert rc == 1 + int(sp.ErrorKind.InvalidArgument)
