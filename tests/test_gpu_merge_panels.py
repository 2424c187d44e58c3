"""GPU parity: the column-panelled merge engine (x larger than the L2 -> K column panels).

The panel count is chosen from 8n at build time (K = ceil(8n / 64 MiB), at most 16); here
SPMVLAB_MERGE_PANELS forces K on small matrices so the panel paths (stacked panel CRS, per-panel
merge tiles, accumulating kernels, per-panel carry fix-ups) are checked against the oracle at
sizes it finishes in seconds.  The full-size configs 3-5 pick K > 1 by themselves
(test_gpu_fullsize_cfg34.py, test_gpu_fullsize_cfg5.py).
"""
import numpy as np
import pytest
import torch

from matrices import corpus, random_matrix
from parity import assert_y_close

pytestmark = pytest.mark.gpu


def _build(sp, monkeypatch, k, m, n, r, c, v, alg=2):
    monkeypatch.setenv("SPMVLAB_MERGE_PANELS", str(k))
    f = sp.build_format(alg, sp.TripletMatrix.from_host(m, n, r, c, v), 1)
    monkeypatch.delenv("SPMVLAB_MERGE_PANELS")
    return f


def _panels_ref(m, n, k, r, c):
    """The panel row pointers and row ids restated in numpy (panel of column c = c // ceil(n / k)):
    panel 0 over all m rows; a panel >= 1 with entries in at most half of the rows doubly
    compressed (only those rows, plus an end entry), the others with their full pointer; offsets
    are into the panel-major element arrays."""
    w = (n + k - 1) // k
    cnt = np.zeros(k * m, dtype=np.int64)
    np.add.at(cnt, (c.astype(np.int64) // w) * m + r.astype(np.int64), 1)
    stacked = np.concatenate([[0], np.cumsum(cnt)])
    ptr, rows = [stacked[:m + 1]], [np.zeros(0, np.int64)]
    for q in range(1, k):
        nz = np.nonzero(cnt[q * m:(q + 1) * m])[0]
        if 2 * len(nz) <= m:  # compressed
            rows.append(nz)
            ptr.append(np.concatenate([stacked[q * m + nz], [stacked[(q + 1) * m]]]))
        else:                 # rows in more than half: the full pointer
            ptr.append(stacked[q * m:(q + 1) * m + 1])
    return np.concatenate(ptr).astype(np.uint32), np.concatenate(rows).astype(np.uint32)


@pytest.mark.parametrize("k", [2, 3, 4, 9, 16])
def test_panels_corpus(cuda, oracle, monkeypatch, k):
    sp = cuda
    for (m, n, r, c, v) in corpus(30, seed=31 + k):
        ref = oracle.build(0, m, n, r, c, v)
        x = np.random.default_rng(k).uniform(-1, 1, n)
        y_ref = oracle.spmv(ref, 0, x)
        bound = oracle.abs_spmv(m, r, c, v, x)
        f = _build(sp, monkeypatch, k, m, n, r, c, v)
        for name in ("row_ptr", "col_ind", "data"):  # the reference storage arrays stay bit-exact
            np.testing.assert_array_equal(f.array(name), ref.arrays[name], err_msg=name)
        if len(v) and n >= k:
            want_ptr, want_rows = _panels_ref(m, n, k, r, c)
            np.testing.assert_array_equal(f.array("merge_panel_row_ptr"), want_ptr)
            np.testing.assert_array_equal(f.array("merge_panel_rows"), want_rows)
            # panel arrays: every entry once, panel-major then CRS order
            w = (n + k - 1) // k
            order = np.lexsort((c, r, c // w))
            np.testing.assert_array_equal(f.array("merge_panel_col"), c[order])
            np.testing.assert_array_equal(f.array("merge_panel_data"), v[order])
        y = sp.run_spmv(2, f, torch.from_numpy(x).cuda(), p=4).cpu().numpy()
        assert_y_close(y, y_ref, bound, what=f"panels={k} m={m} n={n}")
        # the other CRS engines on the same format ignore the panels
        np.testing.assert_array_equal(sp.run_spmv(0, f, torch.from_numpy(x).cuda(), p=1).cpu().numpy(), y_ref)


@pytest.mark.parametrize("k", [2, 4, 11])
def test_panels_long_and_empty_rows(cuda, oracle, monkeypatch, k):
    """Rows spanning many tiles in every panel, rows empty in some panels, empty rows, y preset."""
    sp = cuda
    rng = np.random.default_rng(5)
    m, n = 60000, 50000
    rows = [np.full(40000, 3), np.full(25000, 59999), np.full(n // 2, 100)]
    cols = [rng.choice(n, 40000, replace=False), rng.choice(n, 25000, replace=False), np.arange(n // 2)]
    rr = rng.integers(1000, 3000, 8000)
    cc = rng.integers(0, n, 8000)
    key = np.unique(rr.astype(np.int64) * n + cc)
    rows.append(key // n)
    cols.append(key % n)
    r = np.concatenate(rows).astype(np.uint32)
    c = np.concatenate(cols).astype(np.uint32)
    perm = rng.permutation(len(r))
    r, c = r[perm], c[perm]
    v = rng.uniform(-1, 1, len(r))
    x = rng.uniform(-1, 1, n)
    ref = oracle.build(0, m, n, r, c, v)
    y_ref = oracle.spmv(ref, 0, x)
    bound = oracle.abs_spmv(m, r, c, v, x)
    f = _build(sp, monkeypatch, k, m, n, r, c, v)
    y = torch.full((m,), 123.0, dtype=torch.float64, device="cuda")  # y is fully overwritten
    sp.run_spmv(2, f, torch.from_numpy(x).cuda(), y, p=1)
    assert_y_close(y.cpu().numpy(), y_ref, bound, what=f"panels={k} long rows")


@pytest.mark.parametrize("k", [2, 3])
def test_panels_integer_exact(cuda, oracle, monkeypatch, k):
    """test_parallel_spmv.cpp:374-392 with panels: integer data and x = 1 give a bitwise y."""
    sp = cuda
    m, n, r, c, v = random_matrix(3000, 2500, 0.01, seed=3, dense_row_nnz=2500, integer_values=True)
    y_ref = oracle.spmv_triplet(m, r, c, v, np.ones(n))
    f = _build(sp, monkeypatch, k, m, n, r, c, v)
    y = sp.run_spmv(2, f, torch.ones(n, dtype=torch.float64, device="cuda"), p=5).cpu().numpy()
    np.testing.assert_array_equal(y, y_ref)


def test_panel_count_rule(cuda, monkeypatch):
    """Small x: no panels; more panels than columns: none; ParCRS / SeqCrs formats: none."""
    sp = cuda
    m, n, r, c, v = random_matrix(500, 3, 0.5, seed=1)
    f = _build(sp, monkeypatch, 4, m, n, r, c, v)
    with pytest.raises(Exception):
        f.array("merge_panel_row_ptr")
    m, n, r, c, v = random_matrix(400, 400, 0.05, seed=2)
    with pytest.raises(Exception):
        sp.build_format(2, sp.TripletMatrix.from_host(m, n, r, c, v), 1).array("merge_panel_row_ptr")
    with pytest.raises(Exception):
        _build(sp, monkeypatch, 2, m, n, r, c, v, alg=1).array("merge_panel_row_ptr")


def test_panels_iterate(cuda, oracle, monkeypatch):
    """Iterated multiplies over a panelled format track the oracle loop."""
    sp = cuda
    m, n, r, c, v = random_matrix(2000, 2000, 0.01, seed=9)
    v = np.abs(v)
    f = _build(sp, monkeypatch, 3, m, n, r, c, v)
    x0 = torch.from_numpy(np.random.default_rng(1).uniform(0, 1, n)).cuda()
    xs = x0.clone()
    for _ in range(5):
        xs = sp.run_spmv(2, f, xs, p=1)
    xo = x0.cpu().numpy()
    ref = oracle.build(0, m, n, r, c, v)
    for _ in range(5):
        xo = oracle.spmv(ref, 0, xo)
    np.testing.assert_allclose(xs.cpu().numpy(), xo, rtol=1e-12 * 5, atol=0)
