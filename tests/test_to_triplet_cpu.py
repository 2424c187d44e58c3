"""CPU tests: the format -> triplet decoders (crs_to_triplet crs.hpp:94-105, csb_to_triplet
csb.hpp:103-120, mergeb_to_triplet mergeb.hpp:110-127, bcoh_to_triplet bcoh.hpp:379-392) as
restated in oracle/spmv_oracle.c (orc_format_to_triplet), pinned to the reference's own decoders
(oracle/_ref) on the seeded corpus for every format, and the round trip back to the input entries."""
import numpy as np

from matrices import corpus


def test_to_triplet_vs_reference(oracle, reference):
    for i, (m, n, r, c, v) in enumerate(corpus(10, seed=777)):
        key_in = np.sort(r.astype(np.uint64) << 32 | c)
        for alg in range(11):
            for p, l2 in ((1, 512 * 1024), (3, 512)):
                bo = oracle.build(alg, m, n, r, c, v, threads=p, l2_bytes=l2)
                br = reference.build(alg, m, n, r, c, v, threads=p, l2_bytes=l2)
                got = oracle.to_triplet(bo)
                want = reference.to_triplet(br)
                for g, w, what in zip(got, want, ("rows", "cols", "vals")):
                    np.testing.assert_array_equal(g, w, err_msg=f"{i} alg {alg} p {p} {what}")
                # round trip: the same entries as the input
                order = np.argsort(got[0].astype(np.uint64) << 32 | got[1])
                np.testing.assert_array_equal((got[0].astype(np.uint64) << 32 | got[1])[order], key_in)
                src = np.argsort(r.astype(np.uint64) << 32 | c)
                np.testing.assert_array_equal(got[2][order], v[src])
