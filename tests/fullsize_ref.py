"""Independent full-size restatement of the format layouts in torch (TEST INFRASTRUCTURE).

Every conversion in the reference is "sort by a documented unique key, then populate"
(PAPER.md:295).  For matrices too large for the C oracle this module recomputes each format's
storage arrays directly from those documented keys with vectorised torch ops on the GPU:

  CRS     (row, col)                                         inc/crs.hpp:67-91
  CSB     (br, bc, Morton | Hilbert rank in block)           inc/csb.hpp:51-100
  MergeB  (br, bc, in_row, in_col | Hilbert rank in block)   inc/mergeb.hpp:50-108
  BCOH    (band, Hilbert(block), in_row, in_col) | (band, Hilbert(element))   inc/bcoh.hpp:194-376

Hilbert ranks use the classic rotate formulation (the inverse of tests/oracles.hpp:140-159,
x = column, y = row) -- a different algorithm from the library's orientation automaton.
"""
from __future__ import annotations

import numpy as np
import torch


def morton(r: torch.Tensor, c: torch.Tensor, level: int) -> torch.Tensor:
    r, c = r.long(), c.long()
    key = torch.zeros_like(r)
    for b in range(level):
        key |= ((r >> b) & 1) << (2 * b + 1)
        key |= ((c >> b) & 1) << (2 * b)
    return key


def hilbert(r: torch.Tensor, c: torch.Tensor, level: int) -> torch.Tensor:
    """Classic xy2d with x = column, y = row."""
    x, y = c.long().clone(), r.long().clone()
    d = torch.zeros_like(x)
    nside = 1 << level
    s = nside >> 1
    while s > 0:
        rx = ((x & s) > 0).long()
        ry = ((y & s) > 0).long()
        d += s * s * ((3 * rx) ^ ry)
        # rotate the quadrant (using the full side n, as in the classic algorithm)
        flip = (ry == 0) & (rx == 1)
        x = torch.where(flip, nside - 1 - x, x)
        y = torch.where(flip, nside - 1 - y, y)
        swap = ry == 0
        x, y = torch.where(swap, y, x), torch.where(swap, x, y)
        s >>= 1
    return d


def bit_width(v: int) -> int:
    return int(v).bit_length()


def _order(*keys):
    """Indices sorting lexicographically by keys (last key least significant); keys unique."""
    idx = torch.arange(keys[0].numel(), device=keys[0].device)
    for k in reversed(keys):
        _, perm = torch.sort(k[idx], stable=True)
        idx = idx[perm]
    return idx


def crs(m, r, c, v):
    o = _order(r.long(), c.long())
    counts = torch.bincount(r.long(), minlength=m)
    row_ptr = torch.zeros(m + 1, dtype=torch.int64, device=r.device)
    row_ptr[1:] = torch.cumsum(counts, 0)
    return {"row_ptr": row_ptr, "col_ind": c.long()[o], "data": v[o]}


def csb(m, n, r, c, v, lb, hilbert_order):
    beta = 1 << lb
    mask = beta - 1
    br, bc = r.long() >> lb, c.long() >> lb
    ir, ic = r.long() & mask, c.long() & mask
    rank = hilbert(ir, ic, lb) if hilbert_order else morton(ir, ic, lb)
    o = _order(br, bc, rank)
    block_rows, block_cols = (m + beta - 1) >> lb, (n + beta - 1) >> lb
    cell = br * block_cols + bc
    blk_ptr = torch.zeros(block_rows * block_cols + 1, dtype=torch.int64, device=r.device)
    blk_ptr[1:] = torch.cumsum(torch.bincount(cell, minlength=block_rows * block_cols), 0)
    return {"blk_ptr": blk_ptr, "packed": (ir[o] << 16) | ic[o], "data": v[o]}


def mergeb(m, n, r, c, v, lb, hilbert_order):
    beta = 1 << lb
    mask = beta - 1
    br, bc = r.long() >> lb, c.long() >> lb
    ir, ic = r.long() & mask, c.long() & mask
    if hilbert_order:
        o = _order(br, bc, hilbert(ir, ic, lb))
    else:
        o = _order(br, bc, ir, ic)
    block_rows = (m + beta - 1) >> lb
    block_cols = (n + beta - 1) >> lb
    cell = (br * block_cols + bc)[o]
    new = torch.ones_like(cell, dtype=torch.bool)
    new[1:] = cell[1:] != cell[:-1]
    starts = torch.nonzero(new).flatten()
    blk_br = br[o][starts]
    blk_row_ptr = torch.zeros(block_rows + 1, dtype=torch.int64, device=r.device)
    blk_row_ptr[1:] = torch.cumsum(torch.bincount(blk_br, minlength=block_rows), 0)
    blk_data_ptr = torch.cat([starts, torch.tensor([len(o)], device=r.device)])
    return {"blk_row_ptr": blk_row_ptr, "blk_col_ind": bc[o][starts], "blk_data_ptr": blk_data_ptr,
            "packed": (ir[o] << 16) | ic[o], "data": v[o]}


def bcoh(m, n, r, c, v, lb, bounds, variant):
    """variant: 'bcoh' (ICRS, row-wise, BICRS), 'bcohc' (packed, row-wise, BICRS),
    'bcohch' (packed, Hilbert, BICRS), 'bcohchp' (packed, Hilbert, Hilbert pointer)."""
    dev = r.device
    beta = 1 << lb
    mask = beta - 1
    p = len(bounds) - 1
    block_cols = (n + beta - 1) >> lb
    cov = bit_width(max(m, n, 1) - 1)
    element_level = max(cov, lb)
    block_level = element_level - lb
    rl, cl = r.long(), c.long()
    bnd = torch.tensor(bounds, device=dev, dtype=torch.int64)
    band = torch.searchsorted(bnd, rl, right=True) - 1
    br, bc, ir, ic = rl >> lb, cl >> lb, rl & mask, cl & mask
    if variant in ("bcohch", "bcohchp"):
        o = _order(band, hilbert(rl, cl, element_level))
    else:
        o = _order(band, hilbert(br, bc, block_level), ir, ic)
    band, br, bc, ir, ic, vv = band[o], br[o], bc[o], ir[o], ic[o], v[o]
    nnz = len(o)
    fbr = torch.tensor([b >> lb for b in bounds[:-1]], device=dev, dtype=torch.int64)
    out = {"data": vv}
    # element-level
    new_band = torch.ones(nnz, dtype=torch.bool, device=dev)
    new_band[1:] = band[1:] != band[:-1]
    new_block = new_band.clone()
    new_block[1:] |= (br[1:] != br[:-1]) | (bc[1:] != bc[:-1])
    if variant == "bcoh":
        prev_ir = torch.roll(ir, 1)
        prev_ic = torch.roll(ic, 1)
        same_row = ~new_block & (ir == prev_ir)
        col_inc = torch.where(new_block, ic, torch.where(same_row, ic - prev_ic, ic - prev_ic + beta))
        rj_flag = new_block | ~same_row
        row_jump = torch.where(new_block, ir, ir - prev_ir)[rj_flag]
        out.update({"col_inc": col_inc, "row_jump": row_jump, "packed": torch.zeros(0, device=dev)})
    else:
        out.update({"packed": (ir << 16) | ic, "col_inc": torch.zeros(0, device=dev),
                    "row_jump": torch.zeros(0, device=dev)})
    # block-level
    starts = torch.nonzero(new_block).flatten()
    b_band, b_br, b_bc = band[starts], br[starts], bc[starts]
    nb = len(starts)
    if variant != "bcohchp":
        ends = torch.cat([starts[1:], torch.tensor([nnz], device=dev)])
        first = torch.ones(nb, dtype=torch.bool, device=dev)
        first[1:] = b_band[1:] != b_band[:-1]
        pbr, pbc = torch.roll(b_br, 1), torch.roll(b_bc, 1)
        same = ~first & (b_br == pbr)
        cj = torch.where(first, b_bc, torch.where(same, b_bc - pbc, b_bc - pbc + block_cols))
        rjb = torch.where(first, b_br - fbr[b_band], b_br - pbr)[first | ~same]
        out.update({"block_nnz": ends - starts, "col_jump_block": _i16(cj), "row_jump_block": _i16(rjb),
                    "blk_ptr": torch.zeros(0, device=dev)})
    else:
        ptr_parts = []
        counts_cell = {}
        cell_ids = b_br * block_cols + b_bc
        cnt = torch.zeros(((m + beta - 1) >> lb) * block_cols, dtype=torch.int64, device=dev)
        cnt.index_add_(0, cell_ids, (torch.cat([starts[1:], torch.tensor([nnz], device=dev)]) - starts))
        for b in range(p):
            rows_b = 0 if bounds[b + 1] == bounds[b] else ((bounds[b + 1] + beta - 1) >> lb) - (bounds[b] >> lb)
            gr = torch.arange(rows_b, device=dev).repeat_interleave(block_cols) + (bounds[b] >> lb)
            gc = torch.arange(block_cols, device=dev).repeat(rows_b)
            hk = hilbert(gr, gc, block_level)
            order = torch.argsort(hk)
            cc = cnt[(gr * block_cols + gc)[order]]
            ptr_parts.append(torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), torch.cumsum(cc, 0)]))
        out.update({"blk_ptr": torch.cat(ptr_parts), "block_nnz": torch.zeros(0, device=dev),
                    "col_jump_block": torch.zeros(0, device=dev), "row_jump_block": torch.zeros(0, device=dev)})
    return out


def _i16(t: torch.Tensor) -> torch.Tensor:
    """static_cast<int16_t>(static_cast<uint16_t>(v)) for int64 v."""
    return ((t & 0xFFFF) ^ 0x8000) - 0x8000


def as_numpy_like(got: np.ndarray, want: torch.Tensor) -> np.ndarray:
    w = want.cpu().numpy()
    if got.dtype == np.float64:
        return w.astype(np.float64)
    return w.astype(np.int64)


NAMES = {0: "crs", 1: "crs", 2: "crs", 3: "csb", 4: "csbh", 5: "bcoh", 6: "bcohc", 7: "bcohch", 8: "bcohchp",
         9: "mergeb", 10: "mergebh"}


def expected(sp, alg, m, n, r, c, v, lb, p):
    """The storage arrays of engine `alg` (BCOH: p bands) recomputed from the documented keys."""
    if alg <= 2:
        return crs(m, r, c, v)
    if alg in (3, 4):
        return csb(m, n, r, c, v, lb, alg == 4)
    if alg in (9, 10):
        return mergeb(m, n, r, c, v, lb, alg == 10)
    prefix = np.zeros(m + 1, dtype=np.uint64)
    prefix[1:] = np.cumsum(torch.bincount(r.long(), minlength=m).cpu().numpy())
    bounds = sp.partition_rows_by_nnz(prefix.astype(np.uint32), p, lb).tolist()
    return bcoh(m, n, r, c, v, lb, bounds, NAMES[alg])


def assert_format_bit_exact(sp, f, exp, what):
    """Every storage_report array of built format f equals exp[name] bit for bit (on the device)."""
    for a in sp.storage_report(f).arrays:
        got = f.array_device(a.name)
        want = exp[a.name]
        assert got.numel() == want.numel(), (what, a.name, got.numel(), want.numel())
        if got.dtype == torch.float64:
            ok = torch.equal(got.view(torch.int64), want.to(torch.float64).contiguous().view(torch.int64))
        else:
            ok = torch.equal(got, want.to(torch.int64))
        assert ok, f"{what}: {a.name} differs at full size"
        del got, want
