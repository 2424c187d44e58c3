"""CPU tests: the per-format builders with an explicit block size (build_csb csb.hpp:51-57,
build_mergeb mergeb.hpp:50-56, build_bcoh bcoh.hpp:194-205) as restated in oracle/spmv_oracle.c
(orc_build_format_beta), pinned to the reference's own builders (oracle/_ref): every array and y
bitwise equal for block sizes 2 .. 2^8 and several band counts; the reference's argument errors."""
import numpy as np
import pytest

from matrices import corpus
from oracle.oracle import CheckerError


@pytest.mark.parametrize("alg", range(3, 11))
def test_build_beta_vs_reference(oracle, reference, alg):
    for i, (m, n, r, c, v) in enumerate(corpus(8, seed=515)):
        x = oracle.verification_input(n, 3)
        for lb in (1, 2, 4, 8):
            for p in ((1, 3) if 5 <= alg <= 8 else (1,)):
                bo = oracle.build_beta(alg, m, n, r, c, v, lb, p)
                br = reference.build_beta(alg, m, n, r, c, v, lb, p)
                assert bo.storage == br.storage
                for k in br.arrays:
                    np.testing.assert_array_equal(bo.arrays[k], br.arrays[k], err_msg=f"{i} {alg} lb {lb} {k}")
                np.testing.assert_array_equal(oracle.spmv(bo, alg, x, p=p), reference.spmv(br, alg, x, p=p))


def test_build_beta_errors(oracle, reference):
    m, n, r, c, v = corpus(1, seed=3)[-1]
    for alg, lb, p in ((2, 4, 1), (3, 0, 1), (3, 17, 1), (9, 17, 1), (5, 16, 2), (6, 4, 0)):
        with pytest.raises(CheckerError) as e1:
            oracle.build_beta(alg, m, n, r, c, v, lb, p)
        assert e1.value.code == 2  # InvalidArgument
        if lb >= 1:  # make_block_size(0) would be beta = 1: the reference rejects it the same way
            with pytest.raises(CheckerError) as e2:
                reference.build_beta(alg, m, n, r, c, v, lb, p)
            assert e2.value.code == 2
