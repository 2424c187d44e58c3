"""Every merge-CSR tile shape the library instantiates (warp tiles of 32 * {8, 16, 32} merge items,
picked by matrix size at build time, forced here with SPMVLAB_MERGE_IPT) against the C oracle:
y within 1e-12 * sum|a_ij x_j|, integer data bitwise, on matrices with empty rows, long rows
spanning many tiles and a rectangular shape."""
import numpy as np
import pytest
import torch

from parity import assert_y_close

pytestmark = pytest.mark.gpu


def _matrix(seed, m, n, nnz, long_rows=()):
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, m, nnz)
    for lr in long_rows:
        rows[rng.random(nnz) < 0.15] = lr
    cols = rng.integers(0, n, nnz)
    key = np.unique(rows.astype(np.int64) * n + cols)
    return (key // n).astype(np.uint32), (key % n).astype(np.uint32), rng.uniform(-1, 1, len(key))


@pytest.mark.parametrize("ipt", [8, 16, 32])
@pytest.mark.parametrize("shape", [(5000, 5000, 60000, ()), (3000, 7000, 200000, (17, 1500)), (20000, 900, 40000, ())])
def test_merge_tile_shapes(cuda, oracle, monkeypatch, ipt, shape):
    sp = cuda
    m, n, nnz, long_rows = shape
    monkeypatch.setenv("SPMVLAB_MERGE_IPT", str(ipt))
    rows, cols, vals = _matrix(ipt * 7 + m, m, n, nnz, long_rows)
    a = sp.TripletMatrix(m, n, torch.from_numpy(rows.view(np.int32)).cuda(),
                         torch.from_numpy(cols.view(np.int32)).cuda(), torch.from_numpy(vals).cuda())
    f = sp.build_format(2, a, 1)
    assert f.info["merge_ipt"] == ipt
    x = np.random.default_rng(5).uniform(-1, 1, n)
    y = sp.run_spmv(2, f, torch.from_numpy(x).cuda(), p=1).cpu().numpy()
    assert_y_close(y, oracle.spmv_triplet(m, rows, cols, vals, x), oracle.abs_spmv(m, rows, cols, vals, x))
    vi = (rows.astype(np.int64) * 3 + cols) % 7 + 1.0
    ai = sp.TripletMatrix(m, n, a.row_ind, a.col_ind, torch.from_numpy(vi).cuda())
    fi = sp.build_format(2, ai, 1)
    yi = sp.run_spmv(2, fi, torch.ones(n, dtype=torch.float64, device="cuda"), p=1).cpu().numpy()
    np.testing.assert_array_equal(yi, np.bincount(rows, weights=vi, minlength=m))
