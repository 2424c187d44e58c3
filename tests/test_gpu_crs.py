"""GPU parity: CRS conversion (bit-exact), the three CRS engines, merge-path primitives.

Models tests/test_core_formats.cpp:28-111, tests/test_parallel_spmv.cpp:29-192 and
tests/acceptance.cpp:113-227 of the reference.
"""
import numpy as np
import pytest
import torch

from matrices import corpus, e4, random_fast, random_matrix
from parity import assert_y_close

pytestmark = pytest.mark.gpu

CRS_ALGS = (0, 1, 2)


def _dev(sp, m, n, r, c, v):
    return sp.TripletMatrix.from_host(m, n, r, c, v)


def _x(n, seed=5):
    return np.random.default_rng(seed).uniform(-1, 1, n)


def test_e4_all_crs_engines(cuda):
    sp = cuda
    m, n, r, c, v = e4()
    a = _dev(sp, m, n, r, c, v)
    for alg in CRS_ALGS:
        f = sp.build_format(alg, a, 4)
        assert f.array("row_ptr").tolist() == [0, 2, 3, 3, 5]  # test_core_formats.cpp:73-76
        assert f.array("col_ind").tolist() == [0, 2, 1, 0, 3]
        y = sp.run_spmv(alg, f, torch.ones(4, dtype=torch.float64, device="cuda"), p=4)
        assert y.cpu().tolist() == [3.0, 3.0, 0.0, 9.0]


def test_crs_conversion_bit_exact_corpus(cuda, oracle):
    sp = cuda
    for (m, n, r, c, v) in corpus(40):
        ref = oracle.build(0, m, n, r, c, v)
        f = sp.build_format(0, _dev(sp, m, n, r, c, v), 1)
        for name in ("row_ptr", "col_ind", "data"):
            got = f.array(name)
            np.testing.assert_array_equal(got, ref.arrays[name], err_msg=f"{name} m={m} n={n}")
        rep = sp.storage_report(f)
        assert [(a.name, a.bytes) for a in rep.arrays] == ref.storage


def test_crs_engines_corpus(cuda, oracle):
    sp = cuda
    for (m, n, r, c, v) in corpus(40, seed=7):
        ref = oracle.build(0, m, n, r, c, v)
        x = _x(n)
        y_ref = oracle.spmv(ref, 0, x)
        bound = oracle.abs_spmv(m, r, c, v, x)
        f = sp.build_format(2, _dev(sp, m, n, r, c, v), 1)
        xd = torch.from_numpy(x).cuda()
        y_seq = sp.run_spmv(0, f, xd, p=1).cpu().numpy()
        np.testing.assert_array_equal(y_seq, y_ref)  # SeqCrs is bitwise equal (crs.hpp:43-57)
        for alg in (1, 2):
            for p in (1, 3, 8):
                y = sp.run_spmv(alg, f, xd, p=p).cpu().numpy()
                assert_y_close(y, y_ref, bound, what=f"alg {alg} m={m} n={n}")


def test_integer_exact_all_crs_engines(cuda, oracle):
    """tests/test_parallel_spmv.cpp:374-392: integer data, x = 1 -> bitwise equal y."""
    sp = cuda
    m, n, r, c, v = random_matrix(3000, 2500, 0.01, seed=3, dense_row_nnz=2500, integer_values=True)
    y_ref = oracle.spmv_triplet(m, r, c, v, np.ones(n))
    f = sp.build_format(2, _dev(sp, m, n, r, c, v), 1)
    for alg in CRS_ALGS:
        y = sp.run_spmv(alg, f, torch.ones(n, dtype=torch.float64, device="cuda"), p=5).cpu().numpy()
        np.testing.assert_array_equal(y, y_ref)


def test_merge_long_rows_and_empty_rows(cuda, oracle):
    """Rows spanning many CTA tiles (carry fix-up) plus long runs of empty rows."""
    sp = cuda
    rng = np.random.default_rng(11)
    m, n = 50000, 40000
    rows = [np.full(30000, 7), np.full(9000, 8), np.full(20000, 49999)]
    cols = [rng.choice(n, 30000, replace=False), rng.choice(n, 9000, replace=False),
            rng.choice(n, 20000, replace=False)]
    rr = rng.integers(1000, 2000, 5000)
    cc = rng.integers(0, n, 5000)
    key = np.unique(rr.astype(np.int64) * n + cc)
    rows.append(key // n)
    cols.append(key % n)
    r = np.concatenate(rows).astype(np.uint32)
    c = np.concatenate(cols).astype(np.uint32)
    perm = rng.permutation(len(r))
    r, c = r[perm], c[perm]
    v = rng.uniform(-1, 1, len(r))
    x = _x(n)
    ref = oracle.build(0, m, n, r, c, v)
    y_ref = oracle.spmv(ref, 0, x)
    bound = oracle.abs_spmv(m, r, c, v, x)
    f = sp.build_format(2, _dev(sp, m, n, r, c, v), 1)
    y = sp.run_spmv(2, f, torch.from_numpy(x).cuda(), p=1).cpu().numpy()
    assert_y_close(y, y_ref, bound, what="merge long rows")
    y = sp.run_spmv(1, f, torch.from_numpy(x).cuda(), p=1).cpu().numpy()
    assert_y_close(y, y_ref, bound, what="parcrs long rows")
    # SeqCrs long rows go to one CTA each (chunked products, one ordered add chain): still bitwise
    y = sp.run_spmv(0, f, torch.from_numpy(x).cuda(), p=1).cpu().numpy()
    np.testing.assert_array_equal(y, y_ref)
    assert f.array("par_long_rows").tolist() == [7, 8, 49999]


def test_cfg1_er_crs(cuda, oracle):
    """BASELINE configs[0]: ER n=65,536, mean row 16, U[-1,1] values, x U[-1,1]."""
    sp = cuda
    from paper_2502_19284_b200 import gen
    m, n, r, c, v = gen.er_host(65536, 16.0, seed=1)
    x = gen.uniform_x(n, seed=2)
    ref = oracle.build(0, m, n, r, c, v)
    f = sp.build_format(2, _dev(sp, m, n, r, c, v), 1)
    for name in ("row_ptr", "col_ind", "data"):
        np.testing.assert_array_equal(f.array(name), ref.arrays[name])
    y_ref = oracle.spmv(ref, 2, x, p=8)
    bound = oracle.abs_spmv(m, r, c, v, x)
    xd = torch.from_numpy(x).cuda()
    for alg in CRS_ALGS:
        y = sp.run_spmv(alg, f, xd, p=8).cpu().numpy()
        assert_y_close(y, y_ref, bound, what=f"cfg1 alg {alg}")


def test_merge_path_fig3_kat(cuda):
    """tests/test_parallel_spmv.cpp:29-39: A=[1..8], B=[3,3,5,9], 13 path points."""
    sp = cuda
    a = torch.tensor([1, 2, 3, 4, 5, 6, 7, 8], dtype=torch.int32, device="cuda")
    b = torch.tensor([3, 3, 5, 9], dtype=torch.int32, device="cuda")
    expected = [(0, 0), (1, 0), (2, 0), (3, 0), (3, 1), (3, 2), (4, 2), (5, 2), (5, 3), (6, 3), (7, 3),
                (8, 3), (8, 4)]
    diags = torch.arange(13, dtype=torch.int64, device="cuda")
    i = sp.merge_path_search(a, b, diags).cpu().tolist()
    assert [(i[d], d - i[d]) for d in range(13)] == expected


def test_merge_path_random_vs_oracle(cuda, oracle):
    sp = cuda
    rng = np.random.default_rng(23)
    for trial in range(50):
        a = np.cumsum(rng.integers(0, 4, rng.integers(0, 60))).astype(np.uint32)
        b = np.cumsum(rng.integers(0, 4, rng.integers(0, 60))).astype(np.uint32)
        diags = np.arange(len(a) + len(b) + 1)
        got = sp.merge_path_search(torch.from_numpy(a.view(np.int32)).cuda() if len(a) else
                                   torch.zeros(0, dtype=torch.int32, device="cuda"),
                                   torch.from_numpy(b.view(np.int32)).cuda() if len(b) else
                                   torch.zeros(0, dtype=torch.int32, device="cuda"),
                                   torch.from_numpy(diags).cuda()).cpu().numpy()
        want = [oracle.diagonal_search(a, b, int(d))[0] for d in diags]
        np.testing.assert_array_equal(got, want)


def test_radix_sort_and_scan(cuda):
    sp = cuda
    rng = np.random.default_rng(5)
    for n in (1, 17, 4096, 4097, 100000, 1 << 20):
        keys = rng.integers(0, 1 << 62, n, dtype=np.int64)
        keys[: n // 3] = keys[n // 2]  # many equal keys: stability matters
        vals = np.arange(n, dtype=np.int32)
        kd, vd = torch.from_numpy(keys.copy()).cuda(), torch.from_numpy(vals).cuda()
        sp.sort_pairs(kd, vd, 0, 62)
        order = np.argsort(keys, kind="stable")
        np.testing.assert_array_equal(kd.cpu().numpy(), keys[order])
        np.testing.assert_array_equal(vd.cpu().numpy(), vals[order])
        cnt = rng.integers(0, 1000, n).astype(np.int32)
        out = sp.exclusive_scan(torch.from_numpy(cnt).cuda()).cpu().numpy().astype(np.int64)
        np.testing.assert_array_equal(out, np.concatenate([[0], np.cumsum(cnt)]))


def test_radix_sort_unaligned_buffers(cuda):
    """Caller buffers that are not 16-byte aligned take the scalar histogram / value-copy paths."""
    sp = cuda
    rng = np.random.default_rng(8)
    for n in (5, 3071, 3073, 200001):
        keys = rng.integers(0, 1 << 40, n + 1, dtype=np.int64)
        keys[1: n // 4] = keys[n // 2]
        vals = np.arange(n + 1, dtype=np.int32)
        kbuf, vbuf = torch.from_numpy(keys.copy()).cuda(), torch.from_numpy(vals.copy()).cuda()
        kd, vd = kbuf[1:], vbuf[1:]  # 8- and 4-byte offsets from the allocation
        assert kd.data_ptr() % 16 and vd.data_ptr() % 16
        sp.sort_pairs(kd, vd, 0, 40)
        order = np.argsort(keys[1:], kind="stable")
        np.testing.assert_array_equal(kd.cpu().numpy(), keys[1:][order])
        np.testing.assert_array_equal(vd.cpu().numpy(), vals[1:][order])
        assert kbuf[0].item() == keys[0] and vbuf[0].item() == vals[0]


def test_concurrent_streams_share_one_format(cuda, oracle):
    """Formats are immutable and shareable (inc/engine.hpp ownership): multiplies of
    one format on several streams at once must not interfere (per-stream carry scratch)."""
    sp = cuda
    m, n, r, c, v = random_matrix(20000, 20000, 0.002, seed=21, dense_row_nnz=20000)
    bound_x = []
    f = sp.build_format(2, _dev(sp, m, n, r, c, v), 1)
    ref = oracle.build(0, m, n, r, c, v)
    streams = [torch.cuda.Stream() for _ in range(4)]
    xs = [np.random.default_rng(100 + i).uniform(-1, 1, n) for i in range(4)]
    xd = [torch.from_numpy(x).cuda() for x in xs]
    ys = [torch.empty(m, dtype=torch.float64, device="cuda") for _ in range(4)]
    torch.cuda.synchronize()
    for rep in range(5):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                sp.run_spmv(2, f, xd[i], ys[i], p=1, stream=s)
    torch.cuda.synchronize()
    for i in range(4):
        assert_y_close(ys[i].cpu().numpy(), oracle.spmv(ref, 0, xs[i]), oracle.abs_spmv(m, r, c, v, xs[i]),
                       what=f"stream {i}")


def test_errors(cuda):
    sp = cuda
    m, n, r, c, v = e4()
    f = sp.build_format(2, _dev(sp, m, n, r, c, v), 1)
    with pytest.raises(sp.Error) as e:
        sp.run_spmv(2, f, torch.ones(3, dtype=torch.float64, device="cuda"), p=1)
    assert e.value.kind == sp.ErrorKind.DimensionMismatch
    with pytest.raises(sp.Error) as e:
        sp.run_spmv(2, f, torch.ones(4, dtype=torch.float64, device="cuda"), p=0)
    assert e.value.kind == sp.ErrorKind.InvalidArgument
    bad = _dev(sp, 4, 4, np.array([0, 5], np.uint32), np.array([0, 0], np.uint32), np.ones(2))
    with pytest.raises(sp.Error) as e:
        sp.validate(bad)
    assert e.value.kind == sp.ErrorKind.IndexOutOfRange
    dup = _dev(sp, 4, 4, np.array([1, 1], np.uint32), np.array([2, 2], np.uint32), np.ones(2))
    with pytest.raises(sp.Error) as e:
        sp.validate(dup)
    assert e.value.kind == sp.ErrorKind.DuplicateEntry
    with pytest.raises(sp.Error) as e:
        sp.build_format(0, dup, 1)
    assert e.value.kind == sp.ErrorKind.DuplicateEntry
