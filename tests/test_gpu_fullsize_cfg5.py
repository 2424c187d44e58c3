"""Full-size checks at BASELINE configs[4] (R-MAT scale 26, column-normalised, ~1.06 G nonzeros:
indices and offsets near the 32-bit limits, x of 537 MB): the CRS conversion bit-exact against the
torch restatement of its sort key (tests/fullsize_ref.py), every engine's y within 1e-12 *
sum|a_ij x_j|, integer data bitwise, and two iterations of the application loop."""
import pytest
import torch

import fullsize_ref as fr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg5(cuda):
    from paper_2502_19284_b200 import gen
    name, fn = gen.CONFIGS[5]
    m, n, r, c, v = fn("cuda")
    cuda.release_cached_memory()
    yield m, n, r, c, v
    del r, c, v
    cuda.release_cached_memory()


def test_crs_conversion_bit_exact_cfg5(cuda, cfg5):
    sp = cuda
    m, n, r, c, v = cfg5
    f = sp.build_format(2, sp.TripletMatrix(m, n, r, c, v), 1)
    sp.release_cached_memory()  # the build's sort scratch, before torch's own sorts below
    exp = fr.crs(m, r, c, v)
    try:
        fr.assert_format_bit_exact(sp, f, exp, "cfg5 crs")
    finally:
        del f, exp
        sp.release_cached_memory()


def test_engines_full_size_cfg5(cuda, cfg5):
    sp = cuda
    m, n, r, c, v = cfg5
    assert v.numel() > 1_000_000_000
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
    prod = v * x[c.long()]
    y_ref = torch.zeros(m, dtype=torch.float64, device="cuda").index_add_(0, r.long(), prod)
    bound = y_ref.clone()  # v >= 0 and x >= 0: sum|a x| = y
    del prod
    a = sp.TripletMatrix(m, n, r, c, v)
    for alg in (0, 1, 2, 6, 9, 10, 7):
        f = sp.build_format(alg, a, 8)
        y = sp.run_spmv(alg, f, x, p=8)
        assert bool(((y - y_ref).abs() <= 1e-12 * bound).all()), sp.algorithm_name(alg)
        if alg == 2:  # the application loop: two iterations against two reference multiplies
            xi = x.clone()
            sp.iterate(2, f, xi, 2, norms=False)
            y2 = torch.zeros(m, dtype=torch.float64, device="cuda").index_add_(0, r.long(), v * y_ref[c.long()])
            assert bool(((xi - y2).abs() <= 1e-11 * y2.abs() + 1e-300).all())
        del f, y
        sp.release_cached_memory()


def test_integer_exact_cfg5(cuda, cfg5):
    sp = cuda
    m, n, r, c, _ = cfg5
    vi = ((r.long() + 3 * c.long()) % 5 + 1).double()
    want = torch.zeros(m, dtype=torch.float64, device="cuda").index_add_(0, r.long(), vi)
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    a = sp.TripletMatrix(m, n, r, c, vi)
    for alg in (0, 2, 5, 8, 4):
        f = sp.build_format(alg, a, 8)
        ok = bool((sp.run_spmv(alg, f, ones, p=8) == want).all())
        del f
        sp.release_cached_memory()
        assert ok, sp.algorithm_name(alg)
