"""Full-size checks at BASELINE configs[2] (Zipf, n = 2^24, ~90 M nonzeros) and configs[3]
(permuted 5-point Laplacian 4096^2, 84 M nonzeros), where the CPU oracle is too slow:

* every conversion is BIT-EXACT: all storage arrays of all 11 engines equal the arrays recomputed
  from the documented sort keys by the torch restatement (tests/fullsize_ref.py, pinned to the C
  oracle in test_fullsize_ref_cpu.py), compared on the device;
* every engine's y within 1e-12 * sum|a_ij x_j| of an fp64 scatter-add reference;
* integer data with x = 1: every engine bitwise equal to the exact row sums;
* linearity: A(x1 + 2 x2) == A x1 + 2 A x2 within the same normalised bound;
* storage bytes follow the reference's accounting (CRS: 12 nnz + 4 (m + 1)) and the ICRS stream of
  the CRS format decodes back to its coordinates (crs_to_icrs -> bicrs_to_triplet round trip)."""
import pytest
import torch

import fullsize_ref as fr

pytestmark = pytest.mark.gpu

P = 8


@pytest.fixture(scope="module", params=[3, 4], ids=["cfg3_zipf", "cfg4_laplacian"])
def matrix(request, cuda):
    from paper_2502_19284_b200 import gen
    name, fn = gen.CONFIGS[request.param]
    m, n, r, c, v = fn("cuda")
    yield name, m, n, r, c, v
    del r, c, v
    cuda.release_cached_memory()


@pytest.mark.parametrize("alg", [0, 3, 4, 5, 6, 7, 8, 9, 10])
def test_conversion_bit_exact_full_size(cuda, matrix, alg):
    sp = cuda
    name, m, n, r, c, v = matrix
    f = sp.build_format(alg, sp.TripletMatrix(m, n, r, c, v), P)
    exp = fr.expected(sp, alg, m, n, r, c, v, f.info["log2_beta"], P)
    try:
        fr.assert_format_bit_exact(sp, f, exp, f"{name} {fr.NAMES[alg]}")
    finally:
        del f, exp
        sp.release_cached_memory()


def _ref(m, r, c, v, x):
    prod = v * x[c.long()]
    y = torch.zeros(m, dtype=torch.float64, device="cuda").index_add_(0, r.long(), prod)
    b = torch.zeros(m, dtype=torch.float64, device="cuda").index_add_(0, r.long(), prod.abs())
    return y, b


def test_all_engines_full_size(cuda, matrix):
    sp = cuda
    name, m, n, r, c, v = matrix
    g = torch.Generator("cuda").manual_seed(11)
    x1 = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    x2 = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    y1, b1 = _ref(m, r, c, v, x1)
    y2, b2 = _ref(m, r, c, v, x2)
    a = sp.TripletMatrix(m, n, r, c, v)
    for alg in range(11):
        f = sp.build_format(alg, a, P)
        if alg <= 2:
            assert sp.storage_report(f).total() == 12 * v.numel() + 4 * (m + 1)
        z1 = sp.run_spmv(alg, f, x1, p=P)
        assert bool(((z1 - y1).abs() <= 1e-12 * b1).all()), f"{name} {sp.algorithm_name(alg)}"
        z12 = sp.run_spmv(alg, f, x1 + 2 * x2, p=P)
        z2 = sp.run_spmv(alg, f, x2, p=P)
        assert bool(((z12 - (z1 + 2 * z2)).abs() <= 4e-12 * (b1 + 2 * b2)).all()), f"{name} linearity {alg}"
        del f, z1, z2, z12
    torch.cuda.empty_cache()


def test_integer_exact_and_icrs_round_trip(cuda, matrix):
    sp = cuda
    name, m, n, r, c, v = matrix
    vi = ((r.long() * 13 + c.long() * 5) % 7 + 1).double()
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    want = torch.zeros(m, dtype=torch.float64, device="cuda").index_add_(0, r.long(), vi)
    a = sp.TripletMatrix(m, n, r, c, vi)
    for alg in range(11):
        f = sp.build_format(alg, a, P)
        assert bool((sp.run_spmv(alg, f, ones, p=P) == want).all()), f"{name} {sp.algorithm_name(alg)}"
        if alg == 2:
            icrs = sp.crs_to_icrs(f)
            rows, cols = icrs.to_triplet()
            # CRS order: rows non-decreasing, the CRS col_ind, and the same multiset of entries
            rp = torch.from_numpy(f.array("row_ptr").astype("int64")).cuda()
            expect_rows = torch.repeat_interleave(torch.arange(m, device="cuda"), rp[1:] - rp[:-1])
            assert torch.equal(rows.long(), expect_rows)
            ci = torch.from_numpy(f.array("col_ind").view("int32")).cuda()
            assert torch.equal(cols, ci)
            y_icrs, stats = icrs.spmv(ones)
            assert bool((y_icrs == want).all())
            assert stats[1] + 1 == int((rp[1:] > rp[:-1]).sum())  # one row jump per nonempty row
            icrs.close()
        del f
    torch.cuda.empty_cache()
