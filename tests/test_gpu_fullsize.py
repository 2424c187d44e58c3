"""Full-size parity at BASELINE configs[1] (R-MAT scale 22, 65.2M nonzeros) on the GPU.

* Every conversion is BIT-EXACT: all storage_report arrays of all 11 engines equal the arrays
  recomputed from the documented sort keys by the independent torch restatement
  (tests/fullsize_ref.py, itself pinned to the C oracle in test_fullsize_ref_cpu.py).
* Every engine's y is within 1e-12 * sum|a_ij x_j| of a fp64 scatter-add reference.
* With integer values and x = 1 every engine's y is bitwise equal to the exact row sums
  (the reference's integer-exact property, tests/test_parallel_spmv.cpp:374-392)."""
import numpy as np
import pytest
import torch

import fullsize_ref as fr

pytestmark = pytest.mark.gpu

P = 8  # BCOH bands


@pytest.fixture(scope="module")
def cfg2(cuda):
    from paper_2502_19284_b200 import gen
    m, n, r, c, v = gen.rmat_device(22, 16, seed=1)
    return m, n, r, c, v


@pytest.mark.parametrize("alg", [0, 3, 4, 5, 6, 7, 8, 9, 10])
def test_conversion_bit_exact_full_size(cuda, cfg2, alg):
    sp = cuda
    m, n, r, c, v = cfg2
    f = sp.build_format(alg, sp.TripletMatrix(m, n, r, c, v), P)
    exp = fr.expected(sp, alg, m, n, r, c, v, f.info["log2_beta"], P)
    fr.assert_format_bit_exact(sp, f, exp, fr.NAMES[alg])
    del f, exp
    torch.cuda.empty_cache()


def test_all_engines_y_full_size(cuda, cfg2):
    sp = cuda
    m, n, r, c, v = cfg2
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3)) * 2 - 1
    y_ref = torch.zeros(m, dtype=torch.float64, device="cuda")
    y_ref.index_add_(0, r.long(), v * x[c.long()])
    bound = torch.zeros(m, dtype=torch.float64, device="cuda")
    bound.index_add_(0, r.long(), (v * x[c.long()]).abs())
    a = sp.TripletMatrix(m, n, r, c, v)
    for alg in range(11):
        f = sp.build_format(alg, a, P)
        y = sp.run_spmv(alg, f, x, p=P)
        err = (y - y_ref).abs()
        # y_ref itself carries summation error ~ n_row * eps * bound; both within 1e-12 * bound
        assert bool((err <= 1e-12 * bound).all()), f"{sp.algorithm_name(alg)}: max {float((err / bound.clamp_min(1e-300)).max())}"
        del f


def test_seq_crs_bitwise_full_size(cuda, oracle, cfg2):
    """SeqCrs at full size is BITWISE equal to the reference's sequential row sums: the C oracle's
    entry-order spmv_triplet over the (bit-exact) CRS order is the same left-to-right chain."""
    sp = cuda
    m, n, r, c, v = cfg2
    f = sp.build_format(0, sp.TripletMatrix(m, n, r, c, v), 1)
    rp = f.array("row_ptr")
    rows = np.repeat(np.arange(m, dtype=np.uint32), np.diff(rp.astype(np.int64)))
    x = np.random.default_rng(12).uniform(-1, 1, n)
    y = sp.run_spmv(0, f, torch.from_numpy(x).cuda(), p=1).cpu().numpy()
    want = oracle.spmv_triplet(m, rows, f.array("col_ind"), f.array("data"), x)
    np.testing.assert_array_equal(y, want)
    assert len(f.array("par_long_rows")) > 0  # the long-row CTA path ran


def test_integer_exact_full_size(cuda, cfg2):
    sp = cuda
    m, n, r, c, v = cfg2
    vi = ((r.long() * 131 + c.long() * 7) % 5 + 1).double()
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    y_ref = torch.zeros(m, dtype=torch.float64, device="cuda")
    y_ref.index_add_(0, r.long(), vi)
    a = sp.TripletMatrix(m, n, r, c, vi)
    for alg in range(11):
        f = sp.build_format(alg, a, P)
        y = sp.run_spmv(alg, f, ones, p=P)
        assert bool((y == y_ref).all()), sp.algorithm_name(alg)
        del f


@pytest.mark.parametrize("alg", [2, 9, 6, 4])
def test_cfg2_pinned_to_reference(cuda, reference, cfg2, alg):
    """cfg2 pinned directly to the unmodified reference (oracle/_ref, the reference headers compiled
    by oracle/Makefile) built on this box's host cores from the same COO: every storage array of
    CRS (triplet_to_crs, inc/crs.hpp:67-91), MergeB (build_mergeb, inc/mergeb.hpp:50-108), BCOHC
    with p = host threads bands (build_bcoh, inc/bcoh.hpp:194-376) and CSBH (build_csb with the
    Hilbert curve, inc/csb.hpp:51-100) bit for bit; for CRS also y -- merge against the reference's
    spmv_merge within 1e-12 * sum|a_ij x_j|, SeqCrs bitwise against spmv_crs_seq."""
    sp = cuda
    m, n, r, c, v = cfg2
    rows, cols, vals = r.cpu().numpy().view(np.uint32), c.cpu().numpy().view(np.uint32), v.cpu().numpy()
    th = max(1, reference.hardware_threads())
    ref = reference.build(alg, m, n, rows, cols, vals, threads=th, build_threads=th)
    f = sp.build_format(alg, sp.TripletMatrix(m, n, r, c, v), th)
    names = [a.name for a in sp.storage_report(f).arrays]
    assert names == [nm for nm, _ in ref.storage]
    for nm in names:
        got, want = f.array(nm), ref.arrays[nm]
        assert got.shape == want.shape, nm
        if got.dtype == np.float64:
            assert np.array_equal(got.view(np.int64), want.view(np.int64)), nm
        else:
            assert np.array_equal(got.astype(np.int64), want.astype(np.int64)), nm
    if alg == 2:
        x = np.random.default_rng(21).uniform(-1, 1, n)
        xt = torch.from_numpy(x).cuda()
        y = sp.run_spmv(2, f, xt, p=th).cpu().numpy()
        y_ref = reference.spmv(ref, 2, x, p=th)
        rp = f.array("row_ptr").astype(np.int64)
        ri = torch.from_numpy(np.repeat(np.arange(m), np.diff(rp))).cuda()
        prod = (torch.from_numpy(f.array("data")).cuda() *
                xt[torch.from_numpy(f.array("col_ind").astype(np.int64)).cuda()]).abs()
        bound = torch.zeros(m, dtype=torch.float64, device="cuda").index_add_(0, ri, prod).cpu().numpy()
        assert np.all(np.abs(y - y_ref) <= 1e-12 * bound)
        y0 = sp.run_spmv(0, sp.build_format(0, sp.TripletMatrix(m, n, r, c, v), 1), xt, p=1).cpu().numpy()
        ref0 = reference.build(0, m, n, rows, cols, vals, threads=1, build_threads=th)
        np.testing.assert_array_equal(y0, reference.spmv(ref0, 0, x, p=1))
    del f
    torch.cuda.empty_cache()


def test_merge_hot_plan_full_size(cuda, cfg2):
    """The merge engine's hot-x plan at full size (the sampled reference counts of 65.2M entries):
    merge_hot_cols / merge_hot_col bit-exact against the numpy restatement of the selection rule
    (tests/test_gpu_merge_hot.py), and the plan is in use (R-MAT's column skew)."""
    from test_gpu_merge_hot import _hot_ref
    sp = cuda
    m, n, r, c, v = cfg2
    f = sp.build_format(2, sp.TripletMatrix(m, n, r, c, v), 1)
    col = f.array("col_ind")
    want = _hot_ref(n, len(col), col)
    assert want is not None and f.info["merge_hot_slots"] == len(want[0]) > 0
    np.testing.assert_array_equal(f.array("merge_hot_cols"), want[0])
    np.testing.assert_array_equal(f.array("merge_hot_col"), want[1])
    assert abs(f.info["merge_hot_share"] - want[2]) < 1e-12
    assert f.info["merge_hot_share"] > 0.3
