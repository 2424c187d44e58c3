"""GPU parity: spmvlab_cuda_csb_work_items (csrc/csb_items.cu) against the oracle's restatement of
spmv_csb's item list (inc/spmv_parallel.hpp:202-264), whose quadrant leaves are pinned to the
reference's split_block_range in tests/test_csb_items_cpu.py.  Bit-identical lists on seeded skewed
matrices for thresholds from 1 to 2β, and at BASELINE configs[1] (R-MAT scale 22) for the default
threshold 2β and a small one, where the oracle replays the list from the GPU-built blk_ptr / packed
arrays (themselves bit-identical to the reference's, tests/test_gpu_*.py)."""
import numpy as np
import pytest
import torch

from oracle.oracle import Built, CheckerError
from test_csb_items_cpu import CASES, check_structure, skewed

pytestmark = pytest.mark.gpu


def _built_from_gpu(f, alg):
    meta = {k: int(f.info[k]) for k in ("m", "n", "nnz", "log2_beta", "block_rows", "block_cols",
                                         "element_level", "block_level", "bands")}
    meta["alg"] = alg
    arrays = {"blk_ptr": f.array("blk_ptr"), "packed": f.array("packed")}
    return Built(meta, arrays, [])


@pytest.mark.parametrize("alg", [3, 4], ids=["csb", "csbh"])
def test_items_match_oracle(cuda, oracle, alg):
    sp = cuda
    for m, n, nnz, seed in CASES:
        m, n, r, c, v = skewed(m, n, nnz, seed)
        a = sp.TripletMatrix.from_host(m, n, r, c, v)
        for l2 in (4096, 32768):
            f = sp.build_format(alg, a, 4, sp.EngineOptions(l2_bytes=l2))
            bo = oracle.build(alg, m, n, r, c, v, l2_bytes=l2)
            beta = 1 << bo.meta["log2_beta"]
            for thr in (0, 1, 3, 17, beta // 2, 2 * beta, 10 ** 9):
                got = sp.csb_items_numpy(sp.csb_work_items(f, thr))
                want = oracle.csb_work_items(bo, thr)
                assert got.dtype == want.dtype
                np.testing.assert_array_equal(got, want, err_msg=f"alg {alg} l2 {l2} thr {thr}")


def test_items_errors_and_empty(cuda):
    sp = cuda
    m, n, r, c, v = skewed(200, 200, 1000, 4)
    a = sp.TripletMatrix.from_host(m, n, r, c, v)
    with pytest.raises(sp.Error):
        sp.csb_work_items(sp.build_format(2, a, 1))  # not a CSB format
    f = sp.build_format(3, a, 1)
    assert len(sp.csb_items_numpy(sp.csb_work_items(f))) > 0
    e = sp.TripletMatrix.from_host(5, 7, np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0))
    assert sp.csb_work_items(sp.build_format(4, e, 1)).shape[0] == 0


@pytest.mark.parametrize("alg", [3, 4], ids=["csb", "csbh"])
def test_items_full_size_cfg2(cuda, oracle, alg):
    sp = cuda
    from paper_2502_19284_b200 import gen
    name, fn = gen.CONFIGS[2]
    m, n, r, c, v = fn("cuda")
    a = sp.TripletMatrix(m, n, r, c, v)
    f = sp.build_format(alg, a, 8)
    del r, c, v
    bo = _built_from_gpu(f, alg)
    for thr in (0, 2048):
        got = sp.csb_items_numpy(sp.csb_work_items(f, thr))
        want = oracle.csb_work_items(bo, thr)
        np.testing.assert_array_equal(got, want, err_msg=f"{name} thr {thr}")
        check_structure(bo, got, thr)
        assert (got["temp_slot"] >= 0).sum() > 100  # R-MAT: many split block rows
    del f
    torch.cuda.empty_cache()
