"""The input generators' reductions are deterministic and in a documented order
(paper_2502_19284_b200/gen.py): segment_sums is the blocked left-to-right sum (plain left to right
for segments of at most SEG_BLOCK values), so duplicate R-MAT edges are summed exactly as numpy's
unbuffered np.add.at does, and regenerating a matrix reproduces it bit for bit."""
import numpy as np
import pytest
import torch

from paper_2502_19284_b200 import gen


def _blocked(a):
    if len(a) <= gen.SEG_BLOCK:
        t = 0.0
        for i, x in enumerate(a):
            t = x if i == 0 else t + x
        return t
    return _blocked([_blocked(a[i:i + gen.SEG_BLOCK]) for i in range(0, len(a), gen.SEG_BLOCK)])


@pytest.mark.parametrize("maxlen", [0, 1, 7, 32, 33, 100, 1500])
def test_segment_sums_blocked_order(maxlen):
    rng = np.random.default_rng(maxlen)
    counts = rng.integers(0, maxlen + 1, 40)
    counts[::7] = 0
    vals = rng.standard_normal(int(counts.sum())) * 10.0 ** rng.integers(-8, 8, int(counts.sum()))
    got = gen.segment_sums(torch.from_numpy(vals), torch.from_numpy(counts)).numpy()
    starts = np.cumsum(counts) - counts
    want = np.array([_blocked(list(vals[s:s + k])) for s, k in zip(starts, counts)])
    np.testing.assert_array_equal(got, want)


def test_sum_duplicates_matches_add_at():
    rng = np.random.default_rng(3)
    key = rng.integers(0, 500, 20000)  # ~40 duplicates per key: beyond one block for some
    key[:5] = 7
    vals = rng.random(20000)
    uk, sv = gen.sum_duplicates(torch.from_numpy(key), torch.from_numpy(vals))
    u, inv, cnt = np.unique(key, return_inverse=True, return_counts=True)
    want = np.zeros(len(u))
    np.add.at(want, inv, vals)
    np.testing.assert_array_equal(uk.numpy(), u)
    small = cnt <= gen.SEG_BLOCK
    np.testing.assert_array_equal(sv.numpy()[small], want[small])
    np.testing.assert_allclose(sv.numpy(), want, rtol=1e-13)


def test_rmat_device_deterministic_on_cpu():
    a = gen.rmat_device(11, device="cpu", normalize_columns=True)
    b = gen.rmat_device(11, device="cpu", normalize_columns=True)
    for x, y in zip(a[2:], b[2:]):
        assert torch.equal(x.view(torch.int64) if x.dtype == torch.float64 else x,
                           y.view(torch.int64) if y.dtype == torch.float64 else y)
    m, n, r, c, v = a
    colsum = np.zeros(n)
    np.add.at(colsum, c.numpy().astype(np.int64), v.numpy())
    nz = colsum > 0
    np.testing.assert_allclose(colsum[nz], 1.0, rtol=1e-13)
