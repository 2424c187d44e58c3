"""GPU parity: spmvlab_cuda_build_format_beta (build_csb / build_mergeb / build_bcoh at an explicit
block size) against the oracle's builders (pinned to the reference's in tests/test_build_beta_cpu.py):
every storage array bitwise equal and y within 1e-12 * sum|a_ij x_j| for block sizes 2 .. 2^16
(beyond 2^14 the CSB-family multiply leaves the shared-memory window path), band counts 1 and 4;
the reference's argument errors."""
import numpy as np
import pytest
import torch

from matrices import random_fast, random_matrix
from oracle.oracle import CheckerError

pytestmark = pytest.mark.gpu

MATS = [random_matrix(300, 260, 0.03, seed=41, dense_row_nnz=200, leading_empty_rows=True),
        random_fast(40000, 70000, 300000, seed=42)]


@pytest.mark.parametrize("alg", range(3, 11))
def test_build_beta_matches_oracle(cuda, oracle, alg):
    sp = cuda
    for mi, (m, n, r, c, v) in enumerate(MATS):
        a = sp.TripletMatrix.from_host(m, n, r, c, v)
        x = np.random.default_rng(mi).uniform(-1, 1, n)
        xd = torch.from_numpy(x).cuda()
        bound = oracle.abs_spmv(m, r, c, v, x)
        cap = 15 if 5 <= alg <= 8 else 16
        for lb in (1, 2, 5, 9, 14, cap):
            if mi == 0 and lb > 9:
                continue
            for p in ((1, 4) if 5 <= alg <= 8 else (1,)):
                try:
                    ref = oracle.build_beta(alg, m, n, r, c, v, lb, p)
                except CheckerError as e:  # e.g. a BCOH block grid of >= 2^15 columns: Overflow
                    with pytest.raises(sp.Error) as g:
                        sp.build_format_beta(alg, a, lb, p)
                    assert int(g.value.kind) + 1 == e.code
                    continue
                f = sp.build_format_beta(alg, a, lb, p)
                assert f.info["log2_beta"] == lb
                for name, _ in ref.storage:
                    assert np.array_equal(f.array(name), ref.arrays[name]), f"{mi} {alg} lb {lb} p {p}: {name}"
                y = sp.run_spmv(alg, f, xd, p=p).cpu().numpy()
                assert np.all(np.abs(y - oracle.spmv(ref, alg, x, p=p)) <= 1e-12 * bound), f"{mi} {alg} lb {lb}"
                del f


def test_build_beta_errors(cuda):
    sp = cuda
    m, n, r, c, v = MATS[0]
    a = sp.TripletMatrix.from_host(m, n, r, c, v)
    for alg, lb, p in ((2, 4, 1), (3, 0, 1), (3, 17, 1), (10, 17, 1), (5, 16, 2), (7, 4, 0)):
        with pytest.raises(sp.Error) as e:
            sp.build_format_beta(alg, a, lb, p)
        assert e.value.kind == sp.ErrorKind.InvalidArgument
