"""Parity helpers shared by the GPU tests."""
from __future__ import annotations

import numpy as np

# BASELINE.json tolerance: |y - y_ref| <= 1e-12 * sum_j |a_ij * x_j| per entry.
REL_TOL = 1e-12


def assert_y_close(y, y_ref, bound, tol=REL_TOL, what=""):
    y = np.asarray(y)
    y_ref = np.asarray(y_ref)
    assert y.shape == y_ref.shape, (y.shape, y_ref.shape)
    err = np.abs(y - y_ref)
    lim = tol * np.asarray(bound)
    bad = np.nonzero(err > lim)[0]
    if len(bad):
        i = bad[0]
        raise AssertionError(f"{what}: {len(bad)} entries out of tolerance; first row {i}: "
                             f"got {y[i]!r} want {y_ref[i]!r} bound {bound[i]!r}")


def max_norm_err(y, y_ref, bound):
    b = np.asarray(bound)
    e = np.abs(np.asarray(y) - np.asarray(y_ref))
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(b > 0, e / b, np.where(e > 0, np.inf, 0.0))
    return float(r.max()) if r.size else 0.0


def storage_arrays(built):
    """CPU-checker storage list [(name, bytes)]."""
    return list(built.storage)
