"""Generates tests/golden/golden.npz from the REFERENCE ITSELF (oracle/_ref/libspmvref.so, the
unmodified headers of /root/reference compiled by oracle/Makefile).  Run in the dev container:

    make -C oracle && python tests/golden/make_golden.py

The fixture pins the C restatement (oracle/spmv_oracle.c) and, through it, the CUDA library:
curve ranks, block sizes, row partitions, merge-path points, and for a set of small matrices every
storage array of every format plus y (bitwise) for several band / worker counts.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle.oracle import Reference  # noqa: E402
from matrices import e4, random_matrix  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402


def matrices():
    out = {"e4": e4()}
    out["rand_sq"] = random_matrix(97, 97, 0.05, seed=1)
    out["rand_rect"] = random_matrix(61, 143, 0.04, seed=2, leading_empty_rows=True)
    out["dense_row"] = random_matrix(120, 80, 0.02, seed=3, dense_row_nnz=80)
    out["rmat9"] = gen.rmat_host(9, 8, seed=4)
    out["empty"] = (6, 5, np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0))
    return out


def main():
    ref = Reference()
    g = {}
    rng = np.random.default_rng(2026)
    # curves (inc/curves.hpp:107-143)
    for level in (1, 2, 3, 5, 11, 14, 16, 22, 26, 31):
        side = 1 << level
        pts = rng.integers(0, side, size=(64, 2)).astype(np.uint32)
        if level <= 3:
            rr, cc = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
            pts = np.stack([rr.ravel(), cc.ravel()], 1).astype(np.uint32)
        g[f"curve_pts_{level}"] = pts
        g[f"morton_{level}"] = np.array([ref.morton(int(r), int(c), level) for r, c in pts], np.uint64)
        g[f"hilbert_{level}"] = np.array([ref.hilbert(int(r), int(c), level) for r, c in pts], np.uint64)
    # select_block_size (inc/block_size.hpp:47-61)
    bs = []
    for n in (1, 2, 4, 5, 1000, 65536, 1000000, 4194304, 16777216, 67108864, 1 << 31):
        for cap in (15, 16, 12):
            for l2 in (64, 4096, 65536, 512 * 1024, 1 << 40):
                bs.append((n, cap, l2, ref.select_block_size(n, cap, l2)))
    g["block_size"] = np.array(bs, np.uint64)
    # partition_rows_by_nnz (inc/block_size.hpp:73-102)
    parts = []
    for trial in range(40):
        m = int(rng.integers(1, 400))
        counts = rng.integers(0, 50, m)
        if trial % 3 == 0:
            counts[int(rng.integers(0, m))] += 3000
        prefix = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint32)
        p = int(rng.integers(1, 12))
        lb = int(rng.integers(0, 6))
        bounds = ref.partition_rows_by_nnz(prefix, p, lb)
        parts.append((prefix, p, lb, bounds))
    g["partition_count"] = np.array([len(parts)])
    for i, (prefix, p, lb, bounds) in enumerate(parts):
        g[f"partition_{i}_prefix"] = prefix
        g[f"partition_{i}_args"] = np.array([p, lb], np.uint32)
        g[f"partition_{i}_bounds"] = bounds
    # merge path (inc/spmv_parallel.hpp:47-69): Fig. 3 plus random lists
    a = np.arange(1, 9, dtype=np.uint32)
    b = np.array([3, 3, 5, 9], np.uint32)
    g["mp_fig3"] = np.array([ref.diagonal_search(a, b, d) for d in range(13)], np.uint64)
    for i in range(10):
        a = np.cumsum(rng.integers(0, 4, rng.integers(0, 40))).astype(np.uint32)
        b = np.cumsum(rng.integers(0, 4, rng.integers(0, 40))).astype(np.uint32)
        g[f"mp_{i}_a"], g[f"mp_{i}_b"] = a, b
        g[f"mp_{i}_pts"] = np.array([ref.diagonal_search(a, b, d) for d in range(len(a) + len(b) + 1)],
                                    np.uint64).reshape(-1, 2)
    g["verification_input"] = ref.verification_input(32, 1)
    # formats and y
    mats = matrices()
    g["matrix_names"] = np.array(list(mats))
    for name, (m, n, r, c, v) in mats.items():
        g[f"m_{name}_shape"] = np.array([m, n], np.uint32)
        g[f"m_{name}_rows"], g[f"m_{name}_cols"], g[f"m_{name}_vals"] = r, c, v
        x = ref.verification_input(n, 3) if n else np.zeros(0)
        g[f"m_{name}_x"] = x
        for alg in range(11):
            # the format depends on p only for BCOH (band count) and on l2 only for blocked formats
            for p in ((1, 3, 8) if 5 <= alg <= 8 else (1,)):
                for l2 in ((512 * 1024,) if alg <= 2 else (256, 4096, 512 * 1024)):
                    key = f"f_{name}_{alg}_{p}_{l2}"
                    try:
                        built = ref.build(alg, m, n, r, c, v, threads=p, l2_bytes=l2)
                    except Exception as ex:  # record the error kind
                        g[key + "_error"] = np.array([getattr(ex, "code", 100)])
                        continue
                    g[key + "_meta"] = np.array([built.meta[k] for k in
                                                 ("alg", "m", "n", "nnz", "log2_beta", "block_rows", "block_cols",
                                                  "element_level", "block_level", "bands")], np.uint64)
                    g[key + "_storage"] = np.array([b for _, b in built.storage], np.uint64)
                    g[key + "_names"] = np.array([s for s, _ in built.storage])
                    for an, arr in built.arrays.items():
                        g[f"{key}_a_{an}"] = arr
                    # y bitwise; merge-path engines depend on the worker count
                    for py in ((1, 3, 8) if alg in (2, 9, 10) else (p,)):
                        g[f"{key}_y{py}"] = ref.spmv(built, alg, x, p=py)
    out = os.path.join(HERE, "golden.npz")
    np.savez_compressed(out, **g)
    print(out, os.path.getsize(out), "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
