"""GPU parity: spmvlab_cuda_row_prefix (row_counts + row_prefix, inc/triplet.hpp:75-87) bitwise
equal to the oracle's restatement on the seeded corpus and a skewed 1M-entry matrix (rows of one
value meeting inside a warp are counted once per warp); out-of-range rows -> IndexOutOfRange."""
import numpy as np
import pytest

from matrices import corpus, random_fast

pytestmark = pytest.mark.gpu


def test_row_prefix_matches_oracle(cuda, oracle):
    sp = cuda
    rng = np.random.default_rng(5)
    skew = (200000, 3000, np.minimum((200000 * rng.random(1 << 20) ** 4).astype(np.uint32), 199999),
            rng.integers(0, 3000, 1 << 20).astype(np.uint32), np.ones(1 << 20))
    for m, n, r, c, v in corpus(12, seed=808) + [random_fast(50000, 40000, 400000, seed=9), skew]:
        a = sp.TripletMatrix.from_host(m, n, r, c, v)
        got = sp.row_prefix(a).cpu().numpy().view(np.uint32)
        assert np.array_equal(got, oracle.row_prefix(m, r))


def test_row_prefix_out_of_range(cuda):
    sp = cuda
    a = sp.TripletMatrix.from_host(4, 4, np.array([0, 4], np.uint32), np.array([0, 1], np.uint32), np.ones(2))
    with pytest.raises(sp.Error) as e:
        sp.row_prefix(a)
    assert e.value.kind == sp.ErrorKind.IndexOutOfRange
