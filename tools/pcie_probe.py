"""Dev tool: pinned-memory PCIe bandwidth on the GPU box (the floor of bench.py's e2e step)."""
import torch, time
n = 4194304
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timeit(fn, reps=50):
    for _ in range(3): fn()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / reps * 1e3
print("H2D 33.5MB ms", timeit(lambda: d.copy_(h, non_blocking=True)))
print("D2H 33.5MB ms", timeit(lambda: h.copy_(d, non_blocking=True)))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print("H2D||D2H ms", timeit(both))
