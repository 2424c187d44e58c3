"""Standalone ICRS / BICRS on the device against the REFERENCE's own results
(tests/golden/bicrs_golden.json, made by tests/golden/make_bicrs_golden.py from inc/bicrs.hpp):
crs_to_icrs and triplet_to_bicrs arrays bit-exact, bicrs_to_triplet coordinates exact, the
ReplayStats counters exact, y within tolerance (bitwise for integer data), and CorruptFormat for
every corrupted stream the reference rejects.  Models tests/test_core_formats.cpp:106-160."""
import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "bicrs_golden.json")))


def _bits_to_f64(bits):
    return np.array([int(b, 16) for b in bits], dtype=np.uint64).view(np.float64)


def _check_stream(sp, st, want, x, bound, tag):
    arr = st.arrays()
    assert arr["col_inc"].astype(np.int64).tolist() == want["col_inc"], tag
    assert arr["row_jump"].astype(np.int64).tolist() == want["row_jump"], tag
    y, stats = st.spmv(torch.tensor(x, dtype=torch.float64, device="cuda"))
    assert list(stats) == want["stats"], (tag, stats)
    y_ref = _bits_to_f64(want["y_bits"])
    assert np.all(np.abs(y.cpu().numpy() - y_ref) <= 1e-12 * bound), tag
    r, c = st.to_triplet()
    assert r.cpu().numpy().view(np.uint32).tolist() == want["rows"], tag
    assert c.cpu().numpy().view(np.uint32).tolist() == want["cols"], tag


@pytest.mark.parametrize("entry", GOLD, ids=[e["name"] for e in GOLD])
def test_icrs_bicrs_match_reference(cuda, entry):
    sp = cuda
    e = entry
    m, n = e["m"], e["n"]
    rows, cols, vals = np.array(e["rows"], np.uint32), np.array(e["cols"], np.uint32), np.array(e["vals"])
    x = np.array(e["x"])
    bound = np.zeros(m)
    np.add.at(bound, rows.astype(np.int64), np.abs(vals * x[cols.astype(np.int64)]) if len(vals) else 0.0)
    a = sp.TripletMatrix.from_host(m, n, rows, cols, vals)
    f = sp.build_format(0, a, 1)
    icrs = sp.crs_to_icrs(f)
    assert icrs.kind == 0
    _check_stream(sp, icrs, e["icrs"], x, bound, f"{e['name']} icrs")
    for oname, want in e["bicrs"].items():
        order = torch.tensor(want["order"], dtype=torch.int32, device="cuda")
        b = sp.triplet_to_bicrs(a, order)
        assert b.kind == 1
        _check_stream(sp, b, want, x, bound, f"{e['name']} bicrs {oname}")
        np.testing.assert_array_equal(b.arrays()["data"], vals[np.array(want["order"], dtype=np.int64)])
    for cname, want in e["corrupt"].items():
        b = sp.bicrs_from_arrays(m, n, want["col_inc"], want["row_jump"], vals, kind=1)
        with pytest.raises(sp.Error) as err:
            b.spmv(torch.tensor(x, dtype=torch.float64, device="cuda"))
        assert err.value.kind == sp.ErrorKind[want["error"]], (e["name"], cname)
        with pytest.raises(sp.Error):
            b.to_triplet()


def test_icrs_e4_kat_and_errors(cuda):
    """test_core_formats.cpp:106-111 (E4 increments, y = [3,3,0,9]); permutation and length checks."""
    sp = cuda
    a = sp.TripletMatrix.from_host(4, 4, [0, 0, 1, 3, 3], [0, 2, 1, 0, 3], [1.0, 2.0, 3.0, 4.0, 5.0])
    icrs = sp.crs_to_icrs(sp.build_format(2, a, 1))
    assert icrs.arrays()["col_inc"].tolist() == [0, 2, 3, 3, 3, 4]
    assert icrs.arrays()["row_jump"].tolist() == [0, 1, 2]
    y, _ = icrs.spmv(torch.ones(4, dtype=torch.float64, device="cuda"))
    assert y.cpu().tolist() == [3.0, 3.0, 0.0, 9.0]
    with pytest.raises(sp.Error) as err:
        sp.triplet_to_bicrs(a, torch.tensor([0, 1, 1, 3, 4], dtype=torch.int32, device="cuda"))
    assert err.value.kind == sp.ErrorKind.InvalidArgument
    with pytest.raises(sp.Error) as err:
        icrs.spmv(torch.ones(3, dtype=torch.float64, device="cuda"))
    assert err.value.kind == sp.ErrorKind.DimensionMismatch
    with pytest.raises(sp.Error) as err:
        sp.bicrs_from_arrays(4, 4, [0, 1], [0], [1.0, 2.0])
    assert err.value.kind == sp.ErrorKind.CorruptFormat


def test_bicrs_large_random_order_round_trip(cuda, oracle):
    """A 262k-entry R-MAT in a random element order: the decode returns every coordinate in that
    order and the multiply matches the oracle; integer data gives bitwise row sums."""
    sp = cuda
    from paper_2502_19284_b200 import gen
    m, n, r, c, v = gen.rmat_host(14, 16, seed=4)
    perm = np.random.default_rng(2).permutation(len(v))
    a = sp.TripletMatrix.from_host(m, n, r, c, v)
    b = sp.triplet_to_bicrs(a, torch.from_numpy(perm.astype(np.int32)).cuda())
    rr, cc = b.to_triplet()
    np.testing.assert_array_equal(rr.cpu().numpy().view(np.uint32), r[perm])
    np.testing.assert_array_equal(cc.cpu().numpy().view(np.uint32), c[perm])
    x = np.random.default_rng(3).uniform(-1, 1, n)
    y, stats = b.spmv(torch.from_numpy(x).cuda())
    y_ref = oracle.spmv_triplet(m, r, c, v, x)
    bound = oracle.abs_spmv(m, r, c, v, x)
    assert np.all(np.abs(y.cpu().numpy() - y_ref) <= 1e-12 * bound)
    changes = int(np.count_nonzero(np.diff(r[perm].astype(np.int64)))) if len(v) else 0
    assert stats == (changes + 1, changes)
    vi = ((r.astype(np.int64) * 3 + c) % 7 + 1).astype(np.float64)
    bi = sp.triplet_to_bicrs(sp.TripletMatrix.from_host(m, n, r, c, vi), torch.from_numpy(perm.astype(np.int32)).cuda())
    yi, _ = bi.spmv(torch.ones(n, dtype=torch.float64, device="cuda"))
    np.testing.assert_array_equal(yi.cpu().numpy(), oracle.spmv_triplet(m, r, c, vi, np.ones(n)))
