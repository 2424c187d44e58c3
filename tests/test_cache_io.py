"""SPMVLAB1 triplet cache (inc/cache_io.hpp:31-91).

CPU: the C oracle's cache_read/cache_write against fixtures written by the REFERENCE's own
cache_write (tests/golden/make_cache_fixtures.py), including its recorded outcomes for malformed
files (bad magic, truncated header/body, duplicates, out-of-range, dimension overflow, a 64-bit
index narrowed to 32 bits).  GPU: the device ingest returns the same triplets / error kinds and
its writer is byte-identical to the reference's."""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CACHE = os.path.join(HERE, "golden", "cache")
EXPECTED = json.load(open(os.path.join(CACHE, "expected.json")))


@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_oracle_cache_read_matches_reference(oracle, name):
    from oracle.oracle import CheckerError
    exp = EXPECTED[name]
    path = os.path.join(CACHE, name)
    if exp["code"]:
        with pytest.raises(CheckerError) as e:
            oracle.cache_read(path)
        assert e.value.code == exp["code"]
    else:
        m, n, r, c, v = oracle.cache_read(path)
        assert (m, n, len(v)) == (exp["m"], exp["n"], exp["nnz"])


def test_oracle_cache_write_is_byte_identical(oracle, tmp_path):
    for name in ("e4.spmvlab1", "rand.spmvlab1", "empty.spmvlab1"):
        m, n, r, c, v = oracle.cache_read(os.path.join(CACHE, name))
        out = str(tmp_path / name)
        oracle.cache_write(out, m, n, r, c, v)
        assert open(out, "rb").read() == open(os.path.join(CACHE, name), "rb").read()


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_gpu_cache_read_matches_reference(cuda, oracle, name):
    sp = cuda
    exp = EXPECTED[name]
    path = os.path.join(CACHE, name)
    if exp["code"]:
        with pytest.raises(sp.Error) as e:
            sp.cache_read(path)
        assert int(e.value.kind) + 1 == exp["code"], (name, e.value)
        return
    a = sp.cache_read(path)
    m, n, r, c, v = oracle.cache_read(path)
    assert (a.m, a.n, a.nnz()) == (m, n, len(v))
    np.testing.assert_array_equal(a.row_ind.cpu().numpy().view(np.uint32), r)
    np.testing.assert_array_equal(a.col_ind.cpu().numpy().view(np.uint32), c)
    np.testing.assert_array_equal(a.data.cpu().numpy(), v)


@pytest.mark.gpu
def test_gpu_cache_write_round_trip_large(cuda, oracle, tmp_path):
    """Multi-chunk streams (> 4M entries) through the pinned double-buffered reader and writer."""
    sp = cuda
    from paper_2502_19284_b200 import gen
    m, n, r, c, v = gen.rmat_device(18, 24, seed=3)
    a = sp.TripletMatrix(m, n, r, c, v)
    out = str(tmp_path / "big.spmvlab1")
    sp.cache_write(out, a)
    b = sp.cache_read(out)
    assert (b.m, b.n, b.nnz()) == (a.m, a.n, a.nnz())
    assert a.nnz() > (1 << 22)
    for x, y in ((a.row_ind, b.row_ind), (a.col_ind, b.col_ind), (a.data, b.data)):
        assert bool((x == y).all())
    # and the reference-format bytes: the oracle writer produces the same file
    out2 = str(tmp_path / "big_oracle.spmvlab1")
    oracle.cache_write(out2, m, n, r.cpu().numpy().view(np.uint32), c.cpu().numpy().view(np.uint32), v.cpu().numpy())
    assert open(out, "rb").read() == open(out2, "rb").read()
