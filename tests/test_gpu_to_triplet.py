"""GPU parity: spmvlab_cuda_format_to_triplet (crs_/csb_/mergeb_/bcoh_to_triplet on the device)
against the oracle's restatement, itself pinned to the reference's decoders in
tests/test_to_triplet_cpu.py: bitwise equal rows, columns and values in storage order for every
format on the seeded corpus; at BASELINE configs[1] (R-MAT scale 22) the size-independent round
trip: every format decodes to exactly the input entries."""
import numpy as np
import pytest
import torch

from matrices import corpus, random_fast

pytestmark = pytest.mark.gpu


def test_to_triplet_matches_oracle(cuda, oracle):
    sp = cuda
    mats = corpus(8, seed=99) + [random_fast(3000, 2500, 60000, seed=3)]
    for i, (m, n, r, c, v) in enumerate(mats):
        a = sp.TripletMatrix.from_host(m, n, r, c, v)
        for alg in range(11):
            for p, l2 in ((1, 512 * 1024), (3, 4096)):
                f = sp.build_format(alg, a, p, sp.EngineOptions(l2_bytes=l2))
                t = sp.format_to_triplet(f)
                want = oracle.to_triplet(oracle.build(alg, m, n, r, c, v, threads=p, l2_bytes=l2))
                got = (t.row_ind.cpu().numpy().view(np.uint32), t.col_ind.cpu().numpy().view(np.uint32),
                       t.data.cpu().numpy())
                for g, w, what in zip(got, want, ("rows", "cols", "vals")):
                    np.testing.assert_array_equal(g, w, err_msg=f"{i} {sp.algorithm_name(alg)} p {p} {what}")


def test_family_checks(cuda):
    sp = cuda
    m, n, r, c, v = random_fast(100, 100, 500, seed=1)
    a = sp.TripletMatrix.from_host(m, n, r, c, v)
    f = sp.build_format(3, a, 1)
    assert sp.csb_to_triplet(f).nnz() == len(v)
    with pytest.raises(sp.Error):
        sp.crs_to_triplet(f)
    e = sp.TripletMatrix.from_host(4, 4, np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0))
    for alg in range(11):
        assert sp.format_to_triplet(sp.build_format(alg, e, 2 if 5 <= alg <= 8 else 1)).nnz() == 0


def _keys(rows, cols):
    return (rows.long() & 0xFFFFFFFF) << 32 | (cols.long() & 0xFFFFFFFF)


def test_round_trip_full_size_cfg2(cuda):
    sp = cuda
    from paper_2502_19284_b200 import gen
    name, fn = gen.CONFIGS[2]
    m, n, r, c, v = fn("cuda")
    a = sp.TripletMatrix(m, n, r, c, v)
    k_in, o_in = torch.sort(_keys(r, c))
    v_in = v[o_in]
    del o_in
    for alg in range(11):
        f = sp.build_format(alg, a, 8)
        t = sp.format_to_triplet(f)
        del f
        k, o = torch.sort(_keys(t.row_ind, t.col_ind))
        assert torch.equal(k, k_in), f"{name} {sp.algorithm_name(alg)} coordinates"
        assert torch.equal(t.data[o], v_in), f"{name} {sp.algorithm_name(alg)} values"
        del t, k, o
        torch.cuda.empty_cache()
