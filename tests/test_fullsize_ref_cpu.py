"""Pins tests/fullsize_ref.py (the vectorised torch restatement used for full-size GPU parity)
against the C oracle on small matrices, on the CPU."""
import numpy as np
import pytest
import torch

import fullsize_ref as fr
from matrices import corpus


def test_hilbert_morton_match_oracle(oracle):
    rng = np.random.default_rng(1)
    for level in (1, 2, 5, 11, 14, 22, 26):
        pts = rng.integers(0, 1 << level, size=(500, 2))
        r = torch.from_numpy(pts[:, 0])
        c = torch.from_numpy(pts[:, 1])
        h = fr.hilbert(r, c, level).numpy()
        mo = fr.morton(r, c, level).numpy()
        for k in range(0, 500, 7):
            assert h[k] == oracle.hilbert(int(pts[k, 0]), int(pts[k, 1]), level)
            assert mo[k] == oracle.morton(int(pts[k, 0]), int(pts[k, 1]), level)


NAMES = {3: "csb", 4: "csbh", 5: "bcoh", 6: "bcohc", 7: "bcohch", 8: "bcohchp", 9: "mergeb", 10: "mergebh"}


def expected_arrays(alg, m, n, r, c, v, lb, bounds):
    if alg <= 2:
        return fr.crs(m, r, c, v)
    if alg in (3, 4):
        return fr.csb(m, n, r, c, v, lb, alg == 4)
    if alg in (9, 10):
        return fr.mergeb(m, n, r, c, v, lb, alg == 10)
    return fr.bcoh(m, n, r, c, v, lb, bounds, NAMES[alg])


@pytest.mark.parametrize("l2", [256, 4096])
def test_restatement_matches_oracle(oracle, l2):
    for (m, n, r, c, v) in corpus(15, seed=77):
        if len(v) == 0:
            continue
        rt, ct, vt = torch.from_numpy(r.astype(np.int64)), torch.from_numpy(c.astype(np.int64)), torch.from_numpy(v)
        for alg in (0, 3, 4, 5, 6, 7, 8, 9, 10):
            p = 3
            ref = oracle.build(alg, m, n, r, c, v, threads=p, l2_bytes=l2)
            lb = ref.meta["log2_beta"]
            bounds = ref.arrays["band_first_row"].tolist() + [m] if alg in range(5, 9) else None
            exp = expected_arrays(alg, m, n, rt, ct, vt, lb, bounds)
            for name, _ in ref.storage:
                got = ref.arrays[name]
                np.testing.assert_array_equal(fr.as_numpy_like(got, exp[name]), got.astype(np.float64)
                                              if got.dtype == np.float64 else got.astype(np.int64),
                                              err_msg=f"alg {alg} {name} m={m} n={n}")
