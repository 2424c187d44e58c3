"""GPU parity: the merge engine's hot-x plan (build_hot_columns + merge_hot_kernel).

On a column-skewed matrix (R-MAT) the build gives the most referenced columns a shared-memory
slot: the plan copy merge_hot_col of col_ind marks their entries 0x80000000 | slot and
merge_hot_cols lists them; the persistent tile kernel reads those x values from shared memory.
The plan arrays are checked bit for bit against a numpy restatement of the selection rule, and y
against the oracle within the BASELINE tolerance -- over slot caps, tile counts, long and empty
rows, the fused-exchange (scatter) epilogue and the iterated loop.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from parity import assert_y_close

pytestmark = pytest.mark.gpu

MERGE = 2
MAX_SLOTS, MIN_REFS, MIN_SHARE = 12288, 32, 0.10


SAMPLE, SAMPLE_FROM = 8, 1 << 24


def _hot_ref(n, nnz, crs_col, cap=MAX_SLOTS):
    """The selection rule of build_hot_columns restated: per-column reference counts over the
    sample (every SAMPLE-th run of 32 consecutive col_ind entries from 2^24 nonzeros on, all
    entries below), clamped at 65535 for the threshold search; the threshold T is the smallest
    sampled count >= ceil(MIN_REFS / stride) such that the columns with count >= T fit in cap; kept
    when they cover MIN_SHARE of the entries (sampled counts times the stride)."""
    samp = SAMPLE if nnz >= SAMPLE_FROM else 1
    k = np.arange(nnz)
    sampled = crs_col[(k >> 5) % samp == 0]
    cnt = np.bincount(sampled.astype(np.int64), minlength=n)
    hist = np.bincount(np.minimum(cnt, 65535), minlength=65536)
    take = refs = thr = 0
    for c in range(65535, (MIN_REFS + samp - 1) // samp - 1, -1):
        if take + hist[c] > cap:
            break
        take += hist[c]
        refs += c * hist[c] * samp
        if hist[c]:
            thr = c
    if thr == 0 or take == 0 or refs < MIN_SHARE * nnz:
        return None
    hot = np.nonzero(cnt >= thr)[0]
    slot = np.full(n, -1, np.int64)
    slot[hot] = np.arange(len(hot))
    s = slot[crs_col.astype(np.int64)]
    remap = np.where(s >= 0, s | 0x80000000, crs_col.astype(np.int64)).astype(np.uint32)
    return hot.astype(np.uint32), remap, refs / nnz


def _build(sp, monkeypatch, m, n, r, c, v, **env):
    for k, val in env.items():
        monkeypatch.setenv(k, str(val))
    f = sp.build_format(MERGE, sp.TripletMatrix.from_host(m, n, r, c, v), 1)
    for k in env:
        monkeypatch.delenv(k)
    return f


def _check(sp, oracle, f, m, n, r, c, v, x, cap=MAX_SLOTS, what=""):
    ref = oracle.build(0, m, n, r, c, v)
    want = _hot_ref(n, len(v), ref.arrays["col_ind"], cap)
    assert want is not None, "the matrix should get a hot-x plan"
    hot, remap, share = want
    assert f.info["merge_hot_slots"] == len(hot)
    assert abs(f.info["merge_hot_share"] - share) < 1e-12
    np.testing.assert_array_equal(f.array("merge_hot_cols"), hot)
    np.testing.assert_array_equal(f.array("merge_hot_col"), remap)
    np.testing.assert_array_equal(f.array("col_ind"), ref.arrays["col_ind"])  # storage untouched
    y = sp.run_spmv(MERGE, f, torch.from_numpy(x).cuda(), p=1).cpu().numpy()
    assert_y_close(y, oracle.spmv(ref, 0, x), oracle.abs_spmv(m, r, c, v, x), what=what)
    return ref


@pytest.mark.parametrize("scale,ef,cap,tiles", [(14, 16, None, None), (15, 8, None, None), (14, 16, 64, None),
                                                (14, 16, 1000, 1), (16, 16, None, 16), (13, 4, None, 3)])
def test_hot_rmat(cuda, oracle, monkeypatch, scale, ef, cap, tiles):
    from paper_2502_19284_b200 import gen
    sp = cuda
    m, n, r, c, v = gen.rmat_host(scale, ef, seed=scale + ef)
    env = {}
    if cap is not None:
        env["SPMVLAB_MERGE_HOT_SLOTS"] = cap
    if tiles is not None:
        env["SPMVLAB_MERGE_HOT_TILES"] = tiles
    f = _build(sp, monkeypatch, m, n, r, c, v, **env)
    x = np.random.default_rng(scale).uniform(-1, 1, n)
    _check(sp, oracle, f, m, n, r, c, v, x, cap or MAX_SLOTS, what=f"rmat s{scale} ef{ef} cap={cap} tiles={tiles}")
    # without the plan the same format gives the same y within tolerance (and ParCRS / SeqCrs
    # on it read the untouched col_ind)
    f0 = _build(sp, monkeypatch, m, n, r, c, v, SPMVLAB_MERGE_HOT=0)
    assert f0.info["merge_hot_slots"] == 0
    ref = oracle.build(0, m, n, r, c, v)
    xd = torch.from_numpy(x).cuda()
    assert_y_close(sp.run_spmv(MERGE, f0, xd, p=1).cpu().numpy(), oracle.spmv(ref, 0, x),
                   oracle.abs_spmv(m, r, c, v, x), what="without the plan")
    np.testing.assert_array_equal(sp.run_spmv(0, f, xd, p=1).cpu().numpy(), oracle.spmv(ref, 0, x))


def test_hot_rectangular(cuda, oracle, monkeypatch):
    """A rectangular matrix (m = 3n, then m = n / 4) with skewed columns: the plan and y."""
    from paper_2502_19284_b200 import gen
    sp = cuda
    _, n, r, c, v = gen.rmat_host(14, 16, seed=41)
    for m in (3 * n, n // 4):
        rr = (r.astype(np.int64) * 2654435761 % m).astype(np.uint32)  # rows spread over m
        key = np.unique(rr.astype(np.int64) * n + c)
        r2, c2 = (key // n).astype(np.uint32), (key % n).astype(np.uint32)
        v2 = np.random.default_rng(m).uniform(-1, 1, len(key))
        f = _build(sp, monkeypatch, m, n, r2, c2, v2, SPMVLAB_MERGE_HOT_TILES=2)
        x = np.random.default_rng(1).uniform(-1, 1, n)
        _check(sp, oracle, f, m, n, r2, c2, v2, x, what=f"m={m} n={n}")


def test_hot_long_and_empty_rows(cuda, oracle, monkeypatch):
    """Hot columns inside rows spanning many tiles, runs of empty rows, rows of one entry."""
    sp = cuda
    rng = np.random.default_rng(11)
    m, n = 70000, 40000
    hotc = rng.choice(n, 300, replace=False)
    rows, cols = [], []
    rows.append(np.full(30000, 5)); cols.append(rng.choice(n, 30000, replace=False))          # long row
    rows.append(np.full(n, 69999)); cols.append(np.arange(n))                                  # full last row
    rr = rng.integers(100, 20000, 60000)                                                       # rows >= 20000 stay empty
    rows.append(rr); cols.append(np.where(rng.random(60000) < 0.7, rng.choice(hotc, 60000), rng.integers(0, n, 60000)))
    rows.append(np.arange(40000, 40500)); cols.append(rng.choice(hotc, 500))                  # single-entry rows
    r = np.concatenate(rows).astype(np.int64)
    c = np.concatenate(cols).astype(np.int64)
    key = np.unique(r * n + c)
    r, c = (key // n).astype(np.uint32), (key % n).astype(np.uint32)
    v = rng.uniform(-1, 1, len(key))
    perm = rng.permutation(len(key))
    r, c, v = r[perm], c[perm], v[perm]
    for tiles in (1, 4, 64):
        f = _build(sp, monkeypatch, m, n, r, c, v, SPMVLAB_MERGE_HOT_TILES=tiles)
        for seed in (1, 2):
            x = np.random.default_rng(seed).uniform(-1, 1, n)
            _check(sp, oracle, f, m, n, r, c, v, x, what=f"tiles={tiles} seed={seed}")


def test_hot_plan_skipped_without_skew(cuda, oracle, monkeypatch):
    """Uniform columns (ER, mean degree 16): no column reaches the reference count, no plan."""
    from paper_2502_19284_b200 import gen
    sp = cuda
    m, n, r, c, v = gen.er_host(1 << 14, 16.0, seed=3)
    f = _build(sp, monkeypatch, m, n, r, c, v)
    assert f.info["merge_hot_slots"] == 0
    assert _hot_ref(n, len(v), oracle.build(0, m, n, r, c, v).arrays["col_ind"]) is None


def test_hot_scatter_epilogue(cuda, oracle, monkeypatch):
    """spmvlab_cuda_run_spmv_scatter on a hot-x plan: y, and every destination buffer receives the
    shard's rows at the row offset (the fused exchange's epilogue, here with local buffers)."""
    from paper_2502_19284_b200 import capi, gen
    sp = cuda
    m, n, r, c, v = gen.rmat_host(14, 16, seed=9)
    f = _build(sp, monkeypatch, m, n, r, c, v, SPMVLAB_MERGE_HOT_TILES=2)
    assert f.info["merge_hot_slots"] > 0
    ref = oracle.build(0, m, n, r, c, v)
    x = np.random.default_rng(4).uniform(-1, 1, n)
    y_ref = oracle.spmv(ref, 0, x)
    xd = torch.from_numpy(x).cuda()
    y = torch.full((m,), np.nan, dtype=torch.float64, device="cuda")
    off, dlen = 1234, m + 5000
    dests = [torch.full((dlen,), -7.0, dtype=torch.float64, device="cuda") for _ in range(3)]
    arr = (C.c_void_p * 3)(*[d.data_ptr() for d in dests])
    rc = capi.load().spmvlab_cuda_run_spmv_scatter(f.handle, xd.data_ptr(), n, y.data_ptr(), m, arr, 3, dlen, off,
                                                   torch.cuda.current_stream().cuda_stream)
    assert rc == 0, capi.load().spmvlab_cuda_last_error()
    torch.cuda.synchronize()
    bound = oracle.abs_spmv(m, r, c, v, x)
    assert_y_close(y.cpu().numpy(), y_ref, bound, what="hot scatter y")
    for d in dests:
        dh = d.cpu().numpy()
        np.testing.assert_array_equal(dh[off:off + m], y.cpu().numpy())
        assert (dh[:off] == -7.0).all() and (dh[off + m:] == -7.0).all()


def test_hot_iterate(cuda, oracle, monkeypatch):
    """The iterated loop (x <- A x, normalised) over a hot-x plan vs the oracle loop."""
    from paper_2502_19284_b200 import gen
    sp = cuda
    m, n, r, c, v = gen.rmat_host(13, 16, seed=21, normalize_columns=True)
    f = _build(sp, monkeypatch, m, n, r, c, v)
    assert f.info["merge_hot_slots"] > 0
    ref = oracle.build(0, m, n, r, c, v)
    x = np.full(n, 1.0 / n)
    xd = torch.from_numpy(x.copy()).cuda()
    out = sp.iterate(MERGE, f, xd, 5, p=1)
    xr = x.copy()
    for _ in range(5):
        xr = oracle.spmv(ref, 0, xr)
    got = (out[0] if isinstance(out, tuple) else out).cpu().numpy()
    np.testing.assert_allclose(got, xr, rtol=1e-11, atol=1e-300)


def _oracle_loop(oracle, ref, x0, iters, normalize):
    x, norms = x0.copy(), []
    for _ in range(iters):
        y = oracle.spmv(ref, 0, x)
        mass = y.sum()
        norms.append((np.abs(y - x).sum(), mass))
        x = y / mass if normalize else y
    return x, np.array(norms)


@pytest.mark.parametrize("graph", [False, True])
def test_hot_fused_rescaled_loop(cuda, oracle, monkeypatch, graph):
    """A rescaled loop without norms runs the mass inside the hot-x multiply (per-CTA product sums,
    the scale updated by the carry fix-up's last block): iterates against the oracle loop and
    against the separate pass (SPMVLAB_ITER_FUSED=0); with norms kept, the loop's pass."""
    from paper_2502_19284_b200 import gen
    sp = cuda
    m, n, r, c, v = gen.rmat_host(14, 16, seed=33, normalize_columns=True)
    f = _build(sp, monkeypatch, m, n, r, c, v, SPMVLAB_MERGE_HOT_TILES=3)
    assert f.info["merge_hot_slots"] > 0
    ref = oracle.build(0, m, n, r, c, v)
    x0 = np.random.default_rng(8).uniform(0.0, 1.0, n) + 1e-3
    x0 /= x0.sum()
    want_x, want = _oracle_loop(oracle, ref, x0, 9, True)
    res = {}
    for fused in ("1", "0"):
        for norms in (False, True):
            monkeypatch.setenv("SPMVLAB_ITER_FUSED", fused)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                x = torch.from_numpy(x0.copy()).cuda()
                _, nb = sp.iterate(MERGE, f, x, 9, normalize=True, norms=norms, graph=graph, stream=st)
            st.synchronize()
            monkeypatch.delenv("SPMVLAB_ITER_FUSED")
            got = x.cpu().numpy()
            np.testing.assert_allclose(got, want_x, rtol=2e-11, atol=1e-300)
            assert abs(got.sum() - 1.0) < 1e-12
            if norms:
                nb = nb.cpu().numpy()
                np.testing.assert_allclose(nb[:, 1], want[:, 1], rtol=1e-11)
                np.testing.assert_allclose(nb[:, 0], want[:, 0], rtol=1e-9)
            res[fused, norms] = got
    np.testing.assert_allclose(res["1", False], res["0", False], rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("fused", ["1", "0"])
def test_loop_scale_drift(cuda, oracle, monkeypatch, fused):
    """Rescaling keeps the stored vector unscaled; when the scale leaves [2^-256, 2^256] (a matrix
    whose iterates grow ~1e8 per step) the stored vector is written back scaled.  Both loop forms
    against the oracle's normalised loop over 40 iterations."""
    from paper_2502_19284_b200 import gen
    sp = cuda
    m, n, r, c, v = gen.rmat_host(13, 16, seed=5)
    v = v * 1e7
    f = _build(sp, monkeypatch, m, n, r, c, v)
    assert f.info["merge_hot_slots"] > 0
    ref = oracle.build(0, m, n, r, c, v)
    x0 = np.random.default_rng(9).uniform(0.0, 1.0, n) + 1e-3
    x0 /= x0.sum()
    want_x, want = _oracle_loop(oracle, ref, x0, 40, True)
    monkeypatch.setenv("SPMVLAB_ITER_FUSED", fused)
    x = torch.from_numpy(x0.copy()).cuda()
    _, nb = sp.iterate(MERGE, f, x, 40, normalize=True, norms=fused == "0")  # no norms: the fused path
    monkeypatch.delenv("SPMVLAB_ITER_FUSED")
    got = x.cpu().numpy()
    assert np.isfinite(got).all()
    np.testing.assert_allclose(got, want_x, rtol=1e-10, atol=1e-300)
    if nb is not None:
        np.testing.assert_allclose(nb.cpu().numpy()[:, 1], want[:, 1], rtol=1e-10)


@pytest.mark.parametrize("case", ["one_column", "all_columns_hot", "hot_and_empty_columns"])
def test_hot_edge_matrices(cuda, oracle, monkeypatch, case):
    """Every entry in one column (a 1-slot plan); every column hot (all of x in shared memory);
    hot columns next to never-referenced ones, with some rows empty."""
    sp = cuda
    rng = np.random.default_rng(17)
    if case == "one_column":
        m, n = 50000, 1000
        r = np.arange(0, m, 2, dtype=np.uint32)
        c = np.full(len(r), 777, dtype=np.uint32)
    elif case == "all_columns_hot":
        m, n = 20000, 4096
        key = np.unique(rng.integers(0, m, 400000).astype(np.int64) * n + rng.integers(0, n, 400000))
        r, c = (key // n).astype(np.uint32), (key % n).astype(np.uint32)
    else:
        m, n = 30000, 60000
        hot = rng.choice(n, 2000, replace=False)
        rows = rng.integers(0, m // 2, 300000)  # rows >= m / 2 stay empty
        cols = np.where(rng.random(300000) < 0.9, rng.choice(hot, 300000), rng.integers(0, n, 300000))
        key = np.unique(rows.astype(np.int64) * n + cols)
        r, c = (key // n).astype(np.uint32), (key % n).astype(np.uint32)
    v = rng.uniform(-1, 1, len(r))
    perm = rng.permutation(len(r))
    r, c, v = r[perm], c[perm], v[perm]
    f = _build(sp, monkeypatch, m, n, r, c, v)
    x = rng.uniform(-1, 1, n)
    _check(sp, oracle, f, m, n, r, c, v, x, what=case)
    if case == "all_columns_hot":
        assert f.info["merge_hot_slots"] == n


def test_hot_concurrent_streams(cuda, oracle, monkeypatch):
    """One hot-x format multiplied on four streams at once (per-stream carry scratch; the persistent
    grids of different streams share the SMs)."""
    from paper_2502_19284_b200 import gen
    sp = cuda
    m, n, r, c, v = gen.rmat_host(14, 16, seed=55)
    f = _build(sp, monkeypatch, m, n, r, c, v)
    assert f.info["merge_hot_slots"] > 0
    ref = oracle.build(0, m, n, r, c, v)
    streams = [torch.cuda.Stream() for _ in range(4)]
    xs = [np.random.default_rng(200 + i).uniform(-1, 1, n) for i in range(4)]
    xd = [torch.from_numpy(x).cuda() for x in xs]
    ys = [torch.empty(m, dtype=torch.float64, device="cuda") for _ in range(4)]
    torch.cuda.synchronize()
    for _ in range(5):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                sp.run_spmv(MERGE, f, xd[i], ys[i], p=1, stream=s)
    torch.cuda.synchronize()
    for i in range(4):
        assert_y_close(ys[i].cpu().numpy(), oracle.spmv(ref, 0, xs[i]), oracle.abs_spmv(m, r, c, v, xs[i]),
                       what=f"stream {i}")
