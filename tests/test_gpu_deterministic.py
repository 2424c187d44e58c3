"""Deterministic builds of the blocked formats (EngineOptions.deterministic): every block row is
owned by one CTA that adds into its rows in a fixed order -- the reference's exclusive rows
(inc/spmv_parallel.hpp:311-350) -- so repeated multiplies give the same bits, for all eight blocked
engines (packed and ICRS in-block streams), while the format arrays stay the reference's."""
import numpy as np
import pytest
import torch

from matrices import corpus, random_matrix
from parity import assert_y_close

pytestmark = pytest.mark.gpu
BLOCKED = [3, 4, 5, 6, 7, 8, 9, 10]


def _build(sp, alg, m, n, r, c, v, p, l2=None):
    opt = sp.EngineOptions(deterministic=True)
    if l2:
        opt.l2_bytes = l2
    return sp.build_format(alg, sp.TripletMatrix.from_host(m, n, r, c, v), p, opt)


@pytest.mark.parametrize("alg", BLOCKED)
def test_deterministic_corpus(cuda, oracle, alg):
    sp = cuda
    p = 3
    for (m, n, r, c, v) in corpus(25, seed=70 + alg):
        ref = oracle.build(alg, m, n, r, c, v, threads=p)
        f = _build(sp, alg, m, n, r, c, v, p)
        for name, _ in ref.storage:  # the reference's arrays, bit for bit
            np.testing.assert_array_equal(f.array(name).astype(np.float64 if name == "data" else np.int64),
                                          ref.arrays[name].astype(np.float64 if name == "data" else np.int64),
                                          err_msg=f"{alg} {name}")
        x = np.random.default_rng(alg).uniform(-1, 1, n)
        y = sp.run_spmv(alg, f, torch.from_numpy(x).cuda(), p=p).cpu().numpy()
        assert_y_close(y, oracle.spmv_triplet(m, r, c, v, x), oracle.abs_spmv(m, r, c, v, x),
                       what=f"deterministic alg {alg} m={m} n={n}")


@pytest.mark.parametrize("alg", BLOCKED)
def test_deterministic_repeats_bitwise(cuda, oracle, alg):
    """A power-law matrix with many equal rows per block step (small beta via l2_bytes): ten
    multiplies, identical bits, within tolerance of the oracle; integer data exact."""
    sp = cuda
    from paper_2502_19284_b200 import gen
    m, n, r, c, v = gen.rmat_host(13, 16, seed=7)
    p = 4
    f = _build(sp, alg, m, n, r, c, v, p, l2=64 * 1024)
    x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).cuda()
    y0 = sp.run_spmv(alg, f, x, p=p)
    for _ in range(9):
        assert torch.equal(sp.run_spmv(alg, f, x, p=p).view(torch.int64), y0.view(torch.int64))
    xh = x.cpu().numpy()
    assert_y_close(y0.cpu().numpy(), oracle.spmv_triplet(m, r, c, v, xh), oracle.abs_spmv(m, r, c, v, xh))
    mi, ni, ri, ci, vi = random_matrix(3000, 2000, 0.01, seed=alg, dense_row_nnz=2000, integer_values=True)
    fi = _build(sp, alg, mi, ni, ri, ci, vi, p)
    yi = sp.run_spmv(alg, fi, torch.ones(ni, dtype=torch.float64, device="cuda"), p=p).cpu().numpy()
    np.testing.assert_array_equal(yi, oracle.spmv_triplet(mi, ri, ci, vi, np.ones(ni)))
