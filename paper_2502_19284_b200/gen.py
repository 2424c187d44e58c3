"""Seeded synthetic matrices for the BASELINE.json configurations.

BASELINE.json names no public dataset (the paper's SuiteSparse matrices are not available here),
so these generators stand in for them with the configs' shapes, sizes and value distributions:

  cfg1  Erdos-Renyi, n = 65,536, row degree ~ Binomial(n, 16/n), columns uniform without
        replacement, values U[-1,1]                               -> er_host / er_device
  cfg2  R-MAT scale 22, edge factor 16, (a,b,c,d) = (.57,.19,.19,.05), duplicates summed,
        self loops kept, edge values U(0,1]                        -> rmat_device
  cfg3  Zipf row degrees, exponent 2.1 on [1, 2^20], n = 2^24, columns uniform without
        replacement, values U[-1,1]                               -> zipf_device
  cfg4  5-point Laplacian on a 4096^2 grid (4 / -1), rows and columns permuted by one seeded
        permutation P (P A P^T)                                   -> laplacian_device
  cfg5  R-MAT scale 26 as cfg2, then each column divided by its column sum -> rmat_device(...,
        normalize_columns=True)

Input synthesis only (not the hot path): device generators use torch's seeded CUDA RNG, and the
resulting COO is shuffled so conversions see unordered triplets.  Every reduction is deterministic
(sorts plus fixed-order segment sums, no floating-point atomics), so two processes -- the two bench
arms, or a test and its committed fixture -- generate bit-identical matrices from the same seed.
"""
from __future__ import annotations

import numpy as np
import torch

RMAT_PROBS = (0.57, 0.19, 0.19, 0.05)


# ------------------------------------------------------------------ host (numpy) generators

def uniform_x(n: int, seed: int = 2, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    return np.random.default_rng(seed).uniform(lo, hi, n)


def _unique_cols_per_row(rng, rows: np.ndarray, n: int) -> np.ndarray:
    """Uniform columns without replacement within each row (redraw collisions)."""
    cols = rng.integers(0, n, len(rows), dtype=np.int64)
    while True:
        key = rows.astype(np.int64) * n + cols
        order = np.argsort(key, kind="stable")
        sk = key[order]
        dup = np.zeros(len(sk), dtype=bool)
        dup[1:] = sk[1:] == sk[:-1]
        if not dup.any():
            return cols
        redo = order[dup]
        cols[redo] = rng.integers(0, n, len(redo), dtype=np.int64)


def er_host(n: int, mean_degree: float = 16.0, seed: int = 1):
    """cfg1: Erdos-Renyi rows, degree ~ Binomial(n, mean/n)."""
    rng = np.random.default_rng(seed)
    deg = rng.binomial(n, mean_degree / n, size=n)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    cols = _unique_cols_per_row(rng, rows, n)
    vals = rng.uniform(-1.0, 1.0, len(rows))
    perm = rng.permutation(len(rows))
    return n, n, rows[perm].astype(np.uint32), cols[perm].astype(np.uint32), vals[perm]


def rmat_host(scale: int, edge_factor: int = 16, probs=RMAT_PROBS, seed: int = 1,
              normalize_columns: bool = False):
    """R-MAT on the host (small scales, for tests)."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    e = edge_factor * n
    rows = np.zeros(e, dtype=np.int64)
    cols = np.zeros(e, dtype=np.int64)
    a, b, c, _ = probs
    for lvl in range(scale):
        u = rng.random(e)
        rbit = (u >= a + b).astype(np.int64)
        cbit = (((u >= a) & (u < a + b)) | (u >= a + b + c)).astype(np.int64)
        rows |= rbit << (scale - 1 - lvl)
        cols |= cbit << (scale - 1 - lvl)
    vals = 1.0 - rng.random(e)  # U(0, 1]
    key = rows * n + cols
    uk, inv = np.unique(key, return_inverse=True)
    sv = np.zeros(len(uk))
    np.add.at(sv, inv, vals)
    r = (uk // n).astype(np.uint32)
    cc = (uk % n).astype(np.uint32)
    if normalize_columns:
        colsum = np.zeros(n)
        np.add.at(colsum, cc, sv)
        sv = sv / colsum[cc]
    perm = rng.permutation(len(uk))
    return n, n, r[perm], cc[perm], sv[perm]


# ------------------------------------------------------------------ device (torch) generators

def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def _shuffle(g, *ts):
    perm = torch.randperm(ts[0].numel(), generator=g, device=ts[0].device)
    return [t[perm] for t in ts]


def _as_u32(t: torch.Tensor) -> torch.Tensor:
    out = t.to(torch.int32).contiguous()
    if out.is_cuda:  # the generators' sort temporaries (tens of GB at scale 26) go back to the driver
        torch.cuda.empty_cache()
    return out


SEG_BLOCK = 32


def _short_sums(vals: torch.Tensor, starts: torch.Tensor, lens: torch.Tensor) -> torch.Tensor:
    """out[i] = vals[starts[i]] + vals[starts[i] + 1] + ... (lens[i] terms, left to right)."""
    out = torch.zeros(starts.numel(), dtype=vals.dtype, device=vals.device)
    ne = torch.nonzero(lens > 0).squeeze(1)
    out[ne] = vals[starts[ne]]
    act = torch.nonzero(lens > 1).squeeze(1)
    k = 1
    while act.numel():
        out[act] = out[act] + vals[starts[act] + k]
        k += 1
        act = act[lens[act] > k]
    return out


def segment_sums(vals: torch.Tensor, counts: torch.Tensor) -> torch.Tensor:
    """Deterministic sums of consecutive segments (counts[i] values each, empty segments give 0):
    left to right within blocks of SEG_BLOCK values, then the block sums the same way, recursively.
    A segment of at most SEG_BLOCK values is the plain left-to-right sum."""
    counts = counts.to(torch.int64)
    while True:
        starts = torch.cumsum(counts, 0) - counts
        if counts.numel() == 0 or int(counts.max()) <= SEG_BLOCK:
            return _short_sums(vals, starts, counts)
        npieces = (counts + SEG_BLOCK - 1) // SEG_BLOCK
        seg = torch.repeat_interleave(torch.arange(counts.numel(), device=counts.device), npieces)
        first_piece = torch.cumsum(npieces, 0) - npieces
        within = torch.arange(seg.numel(), device=counts.device) - first_piece[seg]
        pstart = starts[seg] + within * SEG_BLOCK
        plen = torch.clamp(counts[seg] - within * SEG_BLOCK, max=SEG_BLOCK)
        vals = _short_sums(vals, pstart, plen)
        counts = npieces


def sum_duplicates(key: torch.Tensor, vals: torch.Tensor):
    """(unique sorted keys, summed values): duplicates summed in their original order."""
    sk, order = torch.sort(key, stable=True)
    uk, counts = torch.unique_consecutive(sk, return_counts=True)
    del sk
    return uk, segment_sums(vals[order], counts)


def column_sums(cols: torch.Tensor, vals: torch.Tensor, n: int) -> torch.Tensor:
    """Deterministic per-column sums (entries of a column in their storage order)."""
    _, order = torch.sort(cols, stable=True)
    counts = torch.bincount(cols, minlength=n)
    return segment_sums(vals[order], counts)


def rmat_device(scale: int, edge_factor: int = 16, probs=RMAT_PROBS, seed: int = 1,
                normalize_columns: bool = False, device="cuda"):
    """cfg2 / cfg5: R-MAT, duplicates summed, self loops kept, values U(0,1]."""
    g = _gen(seed, device)
    n = 1 << scale
    e = edge_factor * n
    rows = torch.zeros(e, dtype=torch.int64, device=device)
    cols = torch.zeros(e, dtype=torch.int64, device=device)
    a, b, c, _ = probs
    for lvl in range(scale):
        u = torch.rand(e, generator=g, device=device)
        rbit = (u >= a + b).to(torch.int64)
        cbit = (((u >= a) & (u < a + b)) | (u >= a + b + c)).to(torch.int64)
        rows |= rbit << (scale - 1 - lvl)
        cols |= cbit << (scale - 1 - lvl)
        del u, rbit, cbit
    vals = 1.0 - torch.rand(e, generator=g, device=device, dtype=torch.float64)
    key = rows * n + cols
    del rows, cols
    uk, sv = sum_duplicates(key, vals)
    del key, vals
    r = uk // n
    cc = uk % n
    del uk
    if normalize_columns:
        colsum = column_sums(cc, sv, n)
        sv = sv / colsum[cc]
    r, cc, sv = _shuffle(g, r, cc, sv)
    return n, n, _as_u32(r), _as_u32(cc), sv.contiguous()


def er_device(n: int, mean_degree: float = 16.0, seed: int = 1, device="cuda"):
    g = _gen(seed, device)
    deg = torch.binomial(torch.full((n,), float(n), device=device, dtype=torch.float32),
                         torch.full((n,), mean_degree / n, device=device, dtype=torch.float32),
                         generator=g).to(torch.int64)
    rows = torch.repeat_interleave(torch.arange(n, device=device), deg)
    cols = _unique_cols_device(g, rows, n)
    vals = torch.rand(rows.numel(), generator=g, device=device, dtype=torch.float64) * 2 - 1
    rows, cols, vals = _shuffle(g, rows, cols, vals)
    return n, n, _as_u32(rows), _as_u32(cols), vals.contiguous()


def _unique_cols_device(g, rows: torch.Tensor, n: int) -> torch.Tensor:
    cols = torch.randint(0, n, (rows.numel(),), generator=g, device=rows.device)
    while True:
        key = rows * n + cols
        sk, order = torch.sort(key, stable=True)
        dup = torch.zeros_like(sk, dtype=torch.bool)
        dup[1:] = sk[1:] == sk[:-1]
        redo = order[dup]
        if redo.numel() == 0:
            return cols
        cols[redo] = torch.randint(0, n, (redo.numel(),), generator=g, device=rows.device)


def zipf_device(log2_n: int = 24, exponent: float = 2.1, max_degree: int = 1 << 20, seed: int = 3,
                device="cuda"):
    """cfg3: per-row degree from the truncated discrete power law k^-exponent on [1, max_degree]."""
    g = _gen(seed, device)
    n = 1 << log2_n
    k = torch.arange(1, max_degree + 1, device=device, dtype=torch.float64)
    pmf = k.pow(-exponent)
    cdf = torch.cumsum(pmf, 0)
    cdf /= cdf[-1].clone()
    u = torch.rand(n, generator=g, device=device, dtype=torch.float64)
    deg = torch.searchsorted(cdf, u).clamp_(max=max_degree - 1) + 1
    deg = deg.clamp_(max=n)
    rows = torch.repeat_interleave(torch.arange(n, device=device), deg)
    cols = _unique_cols_device(g, rows, n)
    vals = torch.rand(rows.numel(), generator=g, device=device, dtype=torch.float64) * 2 - 1
    rows, cols, vals = _shuffle(g, rows, cols, vals)
    return n, n, _as_u32(rows), _as_u32(cols), vals.contiguous()


def laplacian_device(side: int = 4096, seed: int = 4, device="cuda"):
    """cfg4: 5-point Laplacian (4 diag, -1 neighbours) on side^2, permuted as P A P^T."""
    g = _gen(seed, device)
    n = side * side
    idx = torch.arange(n, device=device)
    i, j = idx // side, idx % side
    parts_r, parts_c, parts_v = [idx], [idx], [torch.full((n,), 4.0, dtype=torch.float64, device=device)]
    for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        ok = (i + di >= 0) & (i + di < side) & (j + dj >= 0) & (j + dj < side)
        src = idx[ok]
        parts_r.append(src)
        parts_c.append(src + di * side + dj)
        parts_v.append(torch.full((src.numel(),), -1.0, dtype=torch.float64, device=device))
    r = torch.cat(parts_r)
    c = torch.cat(parts_c)
    v = torch.cat(parts_v)
    perm = torch.randperm(n, generator=g, device=device)  # P: old index -> new index
    r, c = perm[r], perm[c]
    r, c, v = _shuffle(g, r, c, v)
    return n, n, _as_u32(r), _as_u32(c), v.contiguous()


CONFIGS = {
    1: ("er_n65536_deg16", lambda dev="cuda": er_device(65536, 16.0, 1, dev)),
    2: ("rmat_s22_ef16", lambda dev="cuda": rmat_device(22, 16, RMAT_PROBS, 1, False, dev)),
    3: ("zipf_n2^24_a2.1", lambda dev="cuda": zipf_device(24, 2.1, 1 << 20, 3, dev)),
    4: ("laplacian5_4096^2_permuted", lambda dev="cuda": laplacian_device(4096, 4, dev)),
    5: ("rmat_s26_ef16_colnorm", lambda dev="cuda": rmat_device(26, 16, RMAT_PROBS, 1, True, dev)),
}
