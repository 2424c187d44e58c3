"""GPU parity for the blocked formats: CSB, CSBH, BCOH, BCOHC, BCOHCH, BCOHCHP, MergeB, MergeBH.

Conversions must be bit-exact with the C oracle (itself pinned to the reference) -- every
storage_report array plus the BCOH band tables -- and y within 1e-12 * sum|a_ij x_j|.
Models tests/test_blocked_formats.cpp:199-419 and tests/test_parallel_spmv.cpp:194-392.
"""
import numpy as np
import pytest
import torch

from matrices import corpus, e4, random_matrix
from parity import assert_y_close

pytestmark = pytest.mark.gpu

BLOCKED = (3, 4, 5, 6, 7, 8, 9, 10)
BCOH = (5, 6, 7, 8)
BCOH_TABLES = ("band_first_row", "band_row_count", "band_first_block_row", "band_block_row_count",
               "off_elem", "off_block", "off_row_jump_block", "off_blk_ptr", "off_row_jump")


def _dev(sp, m, n, r, c, v):
    return sp.TripletMatrix.from_host(m, n, r, c, v)


def _check_format(sp, f, ref, alg, tag):
    rep = sp.storage_report(f)
    assert [(a.name, a.bytes) for a in rep.arrays] == ref.storage, tag
    for name, _ in ref.storage:
        np.testing.assert_array_equal(f.array(name), ref.arrays[name], err_msg=f"{tag} {name}")
    if alg in BCOH:
        for name in BCOH_TABLES:
            np.testing.assert_array_equal(f.array(name).astype(np.uint64),
                                          ref.arrays[name].astype(np.uint64), err_msg=f"{tag} {name}")
    for k in ("log2_beta", "block_rows", "block_cols"):
        assert f.info[k] == ref.meta[k], (tag, k)
    if alg in BCOH:
        for k in ("element_level", "block_level", "bands"):
            assert f.info[k] == ref.meta[k], (tag, k)


def test_e4_blocked_kats(cuda, oracle):
    """E4 with beta = 2: CSB blk_ptr [0,2,3,4,5] (test_blocked_formats.cpp:199-206), MergeB
    blk_row_ptr [0,2,4], blk_col_ind [0,1,0,1] (:284-289), y = [3,3,0,9] for every engine."""
    sp = cuda
    m, n, r, c, v = e4()
    a = _dev(sp, m, n, r, c, v)
    opt = sp.EngineOptions(l2_bytes=64)  # forces beta = 2
    f = sp.build_format(3, a, 1, opt)
    assert f.array("blk_ptr").tolist() == [0, 2, 3, 4, 5]
    f = sp.build_format(9, a, 1, opt)
    assert f.array("blk_row_ptr").tolist() == [0, 2, 4]
    assert f.array("blk_col_ind").tolist() == [0, 1, 0, 1]
    ones = torch.ones(4, dtype=torch.float64, device="cuda")
    for alg in BLOCKED:
        for p in (1, 2, 3):
            f = sp.build_format(alg, a, p, opt)
            ref = oracle.build(alg, m, n, r, c, v, threads=p, l2_bytes=64)
            _check_format(sp, f, ref, alg, f"e4 alg {alg} p {p}")
            y = sp.run_spmv(alg, f, ones, p=p).cpu().tolist()
            assert y == [3.0, 3.0, 0.0, 9.0], (alg, p, y)


@pytest.mark.parametrize("l2", [256, 4096, 512 * 1024])
def test_blocked_corpus_bit_exact_and_y(cuda, oracle, l2):
    sp = cuda
    for i, (m, n, r, c, v) in enumerate(corpus(25, seed=100 + l2 % 97)):
        x = np.random.default_rng(i).uniform(-1, 1, n)
        bound = oracle.abs_spmv(m, r, c, v, x)
        a = _dev(sp, m, n, r, c, v)
        xd = torch.from_numpy(x).cuda()
        for alg in BLOCKED:
            for p in ((1, 3, 8) if alg in BCOH else (4,)):
                tag = f"matrix {i} ({m}x{n}, nnz {len(v)}) alg {alg} p {p} l2 {l2}"
                ref = oracle.build(alg, m, n, r, c, v, threads=p, l2_bytes=l2)
                f = sp.build_format(alg, a, p, sp.EngineOptions(l2_bytes=l2))
                _check_format(sp, f, ref, alg, tag)
                y_ref = oracle.spmv(ref, alg, x, p=p)
                y = sp.run_spmv(alg, f, xd, p=p).cpu().numpy()
                assert_y_close(y, y_ref, bound, what=tag)


def test_blocked_larger_power_law(cuda, oracle):
    """A skewed matrix (dense row, empty leading rows) big enough for multi-chunk blocks."""
    sp = cuda
    from paper_2502_19284_b200 import gen
    m, n, r, c, v = gen.rmat_host(13, 8, seed=5)
    x = np.random.default_rng(3).uniform(-1, 1, n)
    bound = oracle.abs_spmv(m, r, c, v, x)
    a = _dev(sp, m, n, r, c, v)
    xd = torch.from_numpy(x).cuda()
    for alg in BLOCKED:
        p = 8 if alg in BCOH else 1
        for l2 in (16384, 512 * 1024):
            ref = oracle.build(alg, m, n, r, c, v, threads=p, l2_bytes=l2)
            f = sp.build_format(alg, a, p, sp.EngineOptions(l2_bytes=l2))
            _check_format(sp, f, ref, alg, f"rmat13 alg {alg} l2 {l2}")
            y = sp.run_spmv(alg, f, xd, p=p).cpu().numpy()
            assert_y_close(y, oracle.spmv(ref, alg, x, p=p), bound, what=f"rmat13 alg {alg}")


def test_integer_exact_all_engines(cuda, oracle):
    """tests/test_parallel_spmv.cpp:374-392: integer data and x = 1 give bitwise-equal y for every
    engine, whatever the summation order."""
    sp = cuda
    m, n, r, c, v = random_matrix(700, 900, 0.02, seed=9, dense_row_nnz=900, integer_values=True)
    y_ref = oracle.spmv_triplet(m, r, c, v, np.ones(n))
    a = _dev(sp, m, n, r, c, v)
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    for alg in range(11):
        for p in (1, 4):
            f = sp.build_format(alg, a, p, sp.EngineOptions(l2_bytes=8192))
            y = sp.run_spmv(alg, f, ones, p=p).cpu().numpy()
            np.testing.assert_array_equal(y, y_ref, err_msg=f"alg {alg} p {p}")


@pytest.mark.parametrize("window", ["0", "1"])
def test_window_and_reduction_kernels(cuda, oracle, monkeypatch, window):
    """CSB / CSBH / MergeB / MergeBH multiply through both device kernels (shared-memory block-row
    window, forced with SPMVLAB_BLOCKED_WINDOW=1; per-run global reduction with =0), on a matrix
    whose block rows span several window items (split rows add into y, whole rows store)."""
    monkeypatch.setenv("SPMVLAB_BLOCKED_WINDOW", window)
    sp = cuda
    from paper_2502_19284_b200 import gen
    m, n, r, c, v = gen.rmat_host(15, 16, seed=8)
    x = np.random.default_rng(4).uniform(-1, 1, n)
    bound = oracle.abs_spmv(m, r, c, v, x)
    a = _dev(sp, m, n, r, c, v)
    xd = torch.from_numpy(x).cuda()
    vi = ((r.astype(np.int64) * 7 + c) % 5 + 1).astype(np.float64)
    ai = _dev(sp, m, n, r, c, vi)
    exact = oracle.spmv_triplet(m, r, c, vi, np.ones(n))
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    for alg in (3, 4, 9, 10, 7, 8):
        ref = oracle.build(alg, m, n, r, c, v, threads=1, l2_bytes=512 * 1024)
        f = sp.build_format(alg, a, 1, sp.EngineOptions(l2_bytes=512 * 1024))
        _check_format(sp, f, ref, alg, f"window {window} alg {alg}")
        names = [d.name for d in sp.storage_report(f).arrays]
        if window == "1":
            whole = f.array("win_item_whole")
            assert 0 in whole and 1 in whole, "expected both split and whole block rows"
        assert "win_item_chunk" not in names  # plan arrays are not storage
        y = sp.run_spmv(alg, f, xd, p=1).cpu().numpy()
        assert_y_close(y, oracle.spmv(ref, alg, x, p=1), bound, what=f"window {window} alg {alg}")
        fi = sp.build_format(alg, ai, 1, sp.EngineOptions(l2_bytes=512 * 1024))
        np.testing.assert_array_equal(sp.run_spmv(alg, fi, ones, p=1).cpu().numpy(), exact)


@pytest.mark.parametrize("l2", [64, 4096])
def test_bcoh_band_partition_paths(cuda, oracle, l2):
    """The band cuts come from per-rounding-cell counts (few cells) or from the full row prefix
    (beta = 2 on 16k rows: 8k cells); both must reproduce partition_rows_by_nnz exactly."""
    sp = cuda
    from paper_2502_19284_b200 import gen
    m, n, r, c, v = gen.rmat_host(14, 4, seed=12)
    a = _dev(sp, m, n, r, c, v)
    for alg in BCOH:
        for p in (2, 5):
            ref = oracle.build(alg, m, n, r, c, v, threads=p, l2_bytes=l2)
            f = sp.build_format(alg, a, p, sp.EngineOptions(l2_bytes=l2))
            _check_format(sp, f, ref, alg, f"rmat14 alg {alg} p {p} l2 {l2}")


def test_bcoh_band_mismatch(cuda):
    """spmv_parallel.hpp:339-341: BCOH multiply with p != bands is InvalidArgument."""
    sp = cuda
    m, n, r, c, v = e4()
    f = sp.build_format(7, _dev(sp, m, n, r, c, v), 2)
    with pytest.raises(sp.Error) as e:
        sp.run_spmv(7, f, torch.ones(4, dtype=torch.float64, device="cuda"), p=3)
    assert e.value.kind == sp.ErrorKind.InvalidArgument
