"""Seeded small test matrices (unique coordinates, shuffled entry order).

Modelled on the reference's test corpus (tests/oracles.hpp:37-109 and
tests/acceptance.cpp:83-111): the E4 running example, random sparse matrices with optional dense
rows / leading empty rows, rectangular shapes and empty matrices.
"""
from __future__ import annotations

import numpy as np


def e4():
    """(0,0)=1, (0,2)=2, (1,1)=3, (3,0)=4, (3,3)=5 -- tests/oracles.hpp:37-44."""
    return (4, 4, np.array([0, 0, 1, 3, 3], np.uint32), np.array([0, 2, 1, 0, 3], np.uint32),
            np.array([1.0, 2.0, 3.0, 4.0, 5.0]))


def random_matrix(m, n, density=0.05, seed=0, dense_row_nnz=0, leading_empty_rows=False,
                  integer_values=False, signed=False):
    """Random sparse matrix with unique coordinates; entries shuffled."""
    rng = np.random.default_rng(seed)
    first_row = m // 4 if leading_empty_rows else 0
    target = int(density * m * n)
    span_r = max(1, m - first_row)
    coords = set()
    if target:
        # draw in bulk until enough unique coordinates
        while len(coords) < target:
            k = (target - len(coords)) * 2 + 8
            r = first_row + rng.integers(0, span_r, k)
            c = rng.integers(0, n, k)
            for rr, cc in zip(r.tolist(), c.tolist()):
                coords.add((rr, cc))
                if len(coords) >= target:
                    break
    for k in range(min(dense_row_nnz, n)):
        coords.add((0, k))
    coords = sorted(coords)
    rows = np.array([r for r, _ in coords], dtype=np.uint32)
    cols = np.array([c for _, c in coords], dtype=np.uint32)
    if integer_values:
        vals = rng.integers(1, 8, len(coords)).astype(np.float64)
    elif signed:
        vals = rng.uniform(-1.0, 1.0, len(coords))
    else:
        vals = 0.5 + rng.integers(0, 1024, len(coords)) / 1024.0
    order = rng.permutation(len(coords))
    return m, n, rows[order], cols[order], vals[order]


def random_fast(m, n, nnz, seed=0, signed=True):
    """Vectorised unique-coordinate matrix for larger sizes (nnz << m*n)."""
    rng = np.random.default_rng(seed)
    keys = np.unique(rng.integers(0, m * n, int(nnz * 1.1) + 16, dtype=np.int64))
    keys = rng.permutation(keys)[:nnz]
    rows = (keys // n).astype(np.uint32)
    cols = (keys % n).astype(np.uint32)
    vals = rng.uniform(-1.0, 1.0, len(keys)) if signed else rng.uniform(0.5, 1.5, len(keys))
    return m, n, rows, cols, vals


def corpus(count=40, seed=20260809):
    """A randomized corpus in the spirit of tests/acceptance.cpp:83-111: square and
    rectangular shapes, dense rows, empty leading rows, tiny and empty matrices."""
    rng = np.random.default_rng(seed)
    out = [e4()]
    out.append((0, 0, np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0)))
    out.append((5, 7, np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0)))
    out.append((1, 1, np.array([0], np.uint32), np.array([0], np.uint32), np.array([2.5])))
    for i in range(count):
        m = int(rng.integers(1, 300))
        n = int(rng.integers(1, 300))
        dens = float(rng.choice([0.002, 0.01, 0.05, 0.2]))
        dense = int(rng.integers(0, n)) if rng.random() < 0.2 else 0
        out.append(random_matrix(m, n, dens, seed=1000 + i, dense_row_nnz=dense,
                                 leading_empty_rows=bool(rng.random() < 0.3)))
    return out
