"""CPU tests: the CSB work-item list of spmv_csb (inc/spmv_parallel.hpp:202-264) as restated in
oracle/spmv_oracle.c (orc_csb_work_items), pinned to the reference:

* every quadrant leaf equals detail::split_block_range's own leaves (oracle/_ref/ref_csb_leaves),
  for Z-Morton and Hilbert in-block order and thresholds from 1 (recursion down to dim == 1) to 2β;
* the list tiles every non-empty block row's elements in order, temp slots as the reference numbers
  them, every chunk within the threshold;
* the multiply that consumes the items (orc spmv_csb with that threshold) is bitwise equal to the
  reference's for each threshold.
"""
import numpy as np
import pytest

from oracle.oracle import CSB_ITEM_DTYPE


def skewed(m, n, nnz, seed):
    """Power-law-like coordinates crowded into the top-left cells (several cells over threshold)."""
    rng = np.random.default_rng(seed)
    r = np.minimum((m * rng.random(nnz * 3) ** 3).astype(np.int64), m - 1)
    c = np.minimum((n * rng.random(nnz * 3) ** 3).astype(np.int64), n - 1)
    keys = np.unique(r * n + c)
    keys = rng.permutation(keys)[:nnz]
    return m, n, (keys // n).astype(np.uint32), (keys % n).astype(np.uint32), rng.uniform(-1, 1, len(keys))


CASES = [(700, 650, 9000, 1), (300, 900, 6000, 2), (1024, 1024, 20000, 3)]


def check_structure(b, items, threshold):
    meta = b.meta
    bcs = meta["block_cols"]
    blk = b.arrays["blk_ptr"].astype(np.int64)
    thr = threshold or 2 << meta["log2_beta"]
    pos, slot = 0, 0
    rows = {}
    for it in items:
        rows.setdefault(int(it["block_row"]), []).append(it)
    for br in range(meta["block_rows"]):
        rb, re = blk[br * bcs], blk[br * bcs + bcs]
        if rb == re:
            assert br not in rows
            continue
        its = rows[br]
        assert its[0]["elem_begin"] == rb and its[-1]["elem_end"] == re
        for a, z in zip(its, its[1:]):
            assert a["elem_end"] == z["elem_begin"]
        if re - rb <= thr:
            assert len(its) == 1 and its[0]["temp_slot"] == -1
            continue
        for it in its:
            assert it["temp_slot"] == slot
            slot += 1
            span = blk[br * bcs + it["cell_end"]] - blk[br * bcs + it["cell_begin"]]
            if it["cell_end"] - it["cell_begin"] > 1 or span <= thr:
                assert it["elem_begin"] == blk[br * bcs + it["cell_begin"]]
                assert it["elem_end"] == blk[br * bcs + it["cell_end"]]
                assert span <= thr
    assert all(items["elem_end"] > items["elem_begin"])


@pytest.mark.parametrize("alg", [3, 4], ids=["csb", "csbh"])
def test_items_vs_reference_leaves(oracle, reference, alg):
    for m, n, nnz, seed in CASES:
        m, n, r, c, v = skewed(m, n, nnz, seed)
        x = oracle.verification_input(n, 5)
        for l2 in (4096, 32768):
            bo = oracle.build(alg, m, n, r, c, v, l2_bytes=l2)
            br = reference.build(alg, m, n, r, c, v, l2_bytes=l2)
            beta = 1 << bo.meta["log2_beta"]
            bcs = bo.meta["block_cols"]
            for thr in (0, 1, 3, 17, beta // 2, 2 * beta):
                items = oracle.csb_work_items(bo, thr)
                assert items.dtype == CSB_ITEM_DTYPE
                check_structure(bo, items, thr)
                t = thr or 2 * beta
                blk = bo.arrays["blk_ptr"].astype(np.int64)
                cells = items["block_row"].astype(np.int64) * bcs + items["cell_begin"]
                over = (items["cell_end"] - items["cell_begin"] == 1) & (blk[cells + 1] - blk[cells] > t)
                got = np.stack([cells[over], items["elem_begin"][over], items["elem_end"][over]], 1)
                want = reference.csb_leaves(br, t).astype(np.int64)
                np.testing.assert_array_equal(got, want, err_msg=f"alg {alg} l2 {l2} thr {thr}")
                for p in (1, 4):
                    np.testing.assert_array_equal(oracle.spmv(bo, alg, x, p=p, split_threshold=thr),
                                                  reference.spmv(br, alg, x, p=p, split_threshold=thr))


def test_items_errors(oracle):
    m, n, r, c, v = skewed(100, 100, 500, 9)
    b = oracle.build(2, m, n, r, c, v)
    from oracle.oracle import CheckerError
    with pytest.raises(CheckerError):
        oracle.csb_work_items(b)
