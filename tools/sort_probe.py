"""Dev tool: the library's LSD onesweep radix sort vs torch.sort (CUB onesweep) on cfg2-sized
(u64 key, u32 value) pairs; per-pass times from the same device."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402

n = 65_245_320
g = torch.Generator("cuda").manual_seed(1)
k0 = torch.randint(0, 1 << 44, (n,), generator=g, device="cuda", dtype=torch.int64)
v0 = torch.arange(n, device="cuda", dtype=torch.int32)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for bits in (44, 48, 64):
    k, v = k0.clone(), v0.clone()
    ms = t(lambda: sp.sort_pairs(k.copy_(k0), v.copy_(v0), 0, bits))
    passes = (bits + 7) // 8
    print(f"library radix sort (u64 key, u32 value), {bits} bits: {ms:.2f} ms = {passes} passes x {ms / passes:.3f} ms "
          f"(incl. two copies of the inputs)", flush=True)
kc = k0.clone()
ms = t(lambda: torch.sort(kc.copy_(k0), stable=True))
print(f"torch.sort (CUB onesweep, int64 keys -> values + int64 indices), 64 bits: {ms:.2f} ms = 8 passes x {ms/8:.3f} ms",
      flush=True)
ms = t(lambda: k.copy_(k0))
print(f"one copy of the keys: {ms:.3f} ms", flush=True)
