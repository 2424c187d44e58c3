"""Order-sensitive device checksum of a COO (test infrastructure): integer arithmetic only (wrapping
int64), so it is exact and independent of the reduction order."""
import torch


def checksum(r: torch.Tensor, c: torch.Tensor, v: torch.Tensor) -> str:
    i = torch.arange(v.numel(), device=v.device, dtype=torch.int64)
    h = (r.long() & 0xFFFFFFFF) * 0x100000001B3 + (c.long() & 0xFFFFFFFF) * 0x9E3779B97F4A7C15 % (1 << 62)
    h = h ^ v.contiguous().view(torch.int64)
    h = h * (i * 2 + 1)  # position-dependent (odd multiplier)
    h = h ^ (h >> 29)
    return f"{int(h.sum().item()) & 0xFFFFFFFFFFFFFFFF:016x}"
