"""CPU tests: the C restatement (oracle/spmv_oracle.c) pinned to the reference.

1. Against tests/golden/golden.npz, recorded from the reference itself (oracle/_ref, see
   tests/golden/make_golden.py): curve ranks, block sizes, row partitions, merge-path points and,
   for several matrices, every format array and y, bitwise.
2. Against the reference's own known-answer tests (E4, Fig. 3, pack_index, block-size examples,
   curve figures; tests/test_*.cpp cited per case).
3. Against oracle/_ref directly on fresh seeded matrices when it is built (dev container).
"""
import os

import numpy as np
import pytest

from matrices import corpus, e4, random_matrix

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def test_golden_curves(oracle, golden):
    for key in golden.files:
        if not key.startswith("curve_pts_"):
            continue
        level = int(key.split("_")[-1])
        pts = golden[key]
        got_m = [oracle.morton(int(r), int(c), level) for r, c in pts]
        got_h = [oracle.hilbert(int(r), int(c), level) for r, c in pts]
        np.testing.assert_array_equal(np.array(got_m, np.uint64), golden[f"morton_{level}"])
        np.testing.assert_array_equal(np.array(got_h, np.uint64), golden[f"hilbert_{level}"])


def test_golden_block_size(oracle, golden):
    for n, cap, l2, lb in golden["block_size"]:
        assert oracle.select_block_size(int(n), int(cap), int(l2)) == int(lb), (n, cap, l2)


def test_golden_partition(oracle, golden):
    for i in range(int(golden["partition_count"][0])):
        p, lb = golden[f"partition_{i}_args"]
        got = oracle.partition_rows_by_nnz(golden[f"partition_{i}_prefix"], int(p), int(lb))
        np.testing.assert_array_equal(got, golden[f"partition_{i}_bounds"])


def test_golden_merge_path(oracle, golden):
    a = np.arange(1, 9, dtype=np.uint32)
    b = np.array([3, 3, 5, 9], np.uint32)
    got = [oracle.diagonal_search(a, b, d) for d in range(13)]
    np.testing.assert_array_equal(np.array(got, np.uint64), golden["mp_fig3"])
    for i in range(10):
        a, b = golden[f"mp_{i}_a"], golden[f"mp_{i}_b"]
        got = [oracle.diagonal_search(a, b, d) for d in range(len(a) + len(b) + 1)]
        np.testing.assert_array_equal(np.array(got, np.uint64).reshape(-1, 2), golden[f"mp_{i}_pts"])


def test_golden_verification_input(oracle, golden):
    np.testing.assert_array_equal(oracle.verification_input(32, 1), golden["verification_input"])


def test_golden_formats_and_y(oracle, golden):
    checked = 0
    for name in golden["matrix_names"]:
        m, n = (int(t) for t in golden[f"m_{name}_shape"])
        r, c, v = golden[f"m_{name}_rows"], golden[f"m_{name}_cols"], golden[f"m_{name}_vals"]
        x = golden[f"m_{name}_x"]
        for key in golden.files:
            prefix = f"f_{name}_"
            if not (key.startswith(prefix) and key.endswith("_meta")):
                continue
            alg, p, l2 = (int(t) for t in key[len(prefix):-len("_meta")].split("_"))
            base = key[:-len("_meta")]
            built = oracle.build(alg, m, n, r, c, v, threads=p, l2_bytes=l2)
            meta = [built.meta[k] for k in ("alg", "m", "n", "nnz", "log2_beta", "block_rows", "block_cols",
                                            "element_level", "block_level", "bands")]
            np.testing.assert_array_equal(np.array(meta, np.uint64), golden[key], err_msg=base)
            assert [s for s, _ in built.storage] == list(golden[base + "_names"]), base
            np.testing.assert_array_equal(np.array([b for _, b in built.storage], np.uint64),
                                          golden[base + "_storage"], err_msg=base)
            for an, arr in built.arrays.items():
                np.testing.assert_array_equal(arr, golden[f"{base}_a_{an}"], err_msg=f"{base} {an}")
            for yk in golden.files:
                if yk.startswith(base + "_y"):
                    py = int(yk[len(base) + 2:])
                    np.testing.assert_array_equal(oracle.spmv(built, alg, x, p=py), golden[yk], err_msg=yk)
            checked += 1
    assert checked > 200


# ---- the reference's own known-answer tests -------------------------------------------------

def test_kat_e4_formats(oracle):
    m, n, r, c, v = e4()
    crs = oracle.build(0, m, n, r, c, v)
    assert crs.arrays["row_ptr"].tolist() == [0, 2, 3, 3, 5]  # test_core_formats.cpp:73-76
    for alg in range(11):
        b = oracle.build(alg, m, n, r, c, v, threads=2)
        assert oracle.spmv(b, alg, np.ones(4), p=2).tolist() == [3, 3, 0, 9]  # oracles.hpp:37-44
    csb = oracle.build(3, m, n, r, c, v, l2_bytes=64)  # beta = 2
    assert csb.arrays["blk_ptr"].tolist() == [0, 2, 3, 4, 5]  # test_blocked_formats.cpp:199-206
    mb = oracle.build(9, m, n, r, c, v, l2_bytes=64)
    assert mb.arrays["blk_row_ptr"].tolist() == [0, 2, 4]  # test_blocked_formats.cpp:284-289
    assert mb.arrays["blk_col_ind"].tolist() == [0, 1, 0, 1]


def test_kat_curves(oracle):
    """tests/test_curves.cpp:28-52."""
    assert [oracle.morton(0, 0, 1), oracle.morton(0, 1, 1), oracle.morton(1, 0, 1), oracle.morton(1, 1, 1)] == [0, 1, 2, 3]
    assert oracle.morton(2, 0, 2) == 8
    assert [oracle.hilbert(0, 0, 1), oracle.hilbert(1, 0, 1), oracle.hilbert(1, 1, 1), oracle.hilbert(0, 1, 1)] == [0, 1, 2, 3]
    assert oracle.hilbert(2, 0, 2) == 4
    for level in range(1, 7):
        side = 1 << level
        seen = set()
        prev = None
        for d in range(side * side):
            r, c = oracle.hilbert_decode(d, level)
            assert oracle.hilbert(r, c, level) == d
            rm, cm = oracle.morton_decode(d, level)
            assert oracle.morton(rm, cm, level) == d
            seen.add((r, c))
            if prev is not None:
                assert abs(prev[0] - r) + abs(prev[1] - c) == 1  # test_curves.cpp:83-95
            prev = (r, c)
        assert len(seen) == side * side


def test_kat_block_size(oracle):
    """tests/test_blocked_formats.cpp:61-98."""
    assert 1 << oracle.select_block_size(1000000, 16, 524288) == 8192
    assert 1 << oracle.select_block_size(1000000, 15, 1 << 40) == 8192
    assert 1 << oracle.select_block_size(4, 16, 1 << 40) == 16
    assert 1 << oracle.select_block_size(1 << 20, 16, 16) == 2


def test_kat_partition_uniform(oracle):
    """tests/test_blocked_formats.cpp:112-121: uniform rows split symmetrically."""
    m = 8 * 4
    prefix = np.arange(m + 1, dtype=np.uint32)
    assert oracle.partition_rows_by_nnz(prefix, 2, 2).tolist() == [0, 16, 32]


def test_validate(oracle):
    assert oracle.validate(4, 4, [0, 1], [1, 1]) == 0
    assert oracle.validate(4, 4, [0, 4], [1, 1]) == 9  # IndexOutOfRange
    assert oracle.validate(4, 4, [1, 1], [2, 2]) == 10  # DuplicateEntry


def test_integer_exact(oracle):
    m, n, r, c, v = random_matrix(200, 150, 0.05, seed=3, dense_row_nnz=150, integer_values=True)
    y_ref = oracle.spmv_triplet(m, r, c, v, np.ones(n))
    for alg in range(11):
        for p in (1, 3):
            b = oracle.build(alg, m, n, r, c, v, threads=p, l2_bytes=4096)
            np.testing.assert_array_equal(oracle.spmv(b, alg, np.ones(n), p=p), y_ref)


def test_oracle_vs_reference_fresh(oracle, reference):
    """Fresh seeded matrices: every array and y bitwise equal to the reference itself."""
    for i, (m, n, r, c, v) in enumerate(corpus(12, seed=4242)):
        x = oracle.verification_input(n, 9)
        for alg in range(11):
            for p in (1, 5):
                for l2 in (512, 512 * 1024):
                    bo = oracle.build(alg, m, n, r, c, v, threads=p, l2_bytes=l2)
                    br = reference.build(alg, m, n, r, c, v, threads=p, l2_bytes=l2)
                    assert bo.storage == br.storage
                    for k in br.arrays:
                        np.testing.assert_array_equal(bo.arrays[k], br.arrays[k], err_msg=f"{i} {alg} {k}")
                    np.testing.assert_array_equal(oracle.spmv(bo, alg, x, p=p), reference.spmv(br, alg, x, p=p))
