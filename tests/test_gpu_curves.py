"""Device curve keys (spmvlab_cuda_curve_keys: the table-driven Morton / Hilbert encoders of
csrc/common.cuh) against the reference's encoders (inc/curves.hpp:107-143) at levels 1..31:
tests/golden/golden.npz holds points and both ranks recorded from oracle/_ref by
tests/golden/make_golden.py; small levels are also checked exhaustively against the C oracle."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden():
    import os
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz"))


def test_device_curve_keys_golden_levels(cuda, golden):
    sp = cuda
    levels = sorted(int(k.split("_")[-1]) for k in golden.files if k.startswith("curve_pts_"))
    assert levels[0] == 1 and levels[-1] == 31
    for level in levels:
        pts = golden[f"curve_pts_{level}"].astype(np.uint32)
        rows = torch.from_numpy(pts[:, 0].view(np.int32)).cuda()
        cols = torch.from_numpy(pts[:, 1].view(np.int32)).cuda()
        for kind, name in ((0, "morton"), (1, "hilbert")):
            got = sp.curve_keys(kind, rows, cols, level).cpu().numpy().view(np.uint64)
            np.testing.assert_array_equal(got, golden[f"{name}_{level}"], err_msg=f"{name} level {level}")


@pytest.mark.parametrize("level", [1, 2, 3, 4, 5, 6])
def test_device_curve_keys_exhaustive_small_levels(cuda, oracle, level):
    sp = cuda
    side = 1 << level
    rr, cc = np.meshgrid(np.arange(side, dtype=np.uint32), np.arange(side, dtype=np.uint32), indexing="ij")
    rows, cols = rr.ravel(), cc.ravel()
    rt = torch.from_numpy(rows.view(np.int32)).cuda()
    ct = torch.from_numpy(cols.view(np.int32)).cuda()
    m = sp.curve_keys(0, rt, ct, level).cpu().numpy().view(np.uint64)
    h = sp.curve_keys(1, rt, ct, level).cpu().numpy().view(np.uint64)
    np.testing.assert_array_equal(m, [oracle.morton(int(r), int(c), level) for r, c in zip(rows, cols)])
    np.testing.assert_array_equal(h, [oracle.hilbert(int(r), int(c), level) for r, c in zip(rows, cols)])
    assert sorted(h.tolist()) == list(range(side * side))  # a bijection onto the curve positions
