"""Quick timing probe (dev tool): R-MAT scale S, CRS build + the three CRS engines."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
algs = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2]
t = time.time()
m, n, r, c, v = gen.rmat_device(scale)
torch.cuda.synchronize()
print(f"gen scale {scale}: nnz={v.numel()} {time.time() - t:.2f}s", flush=True)
a = sp.TripletMatrix(m, n, r, c, v)
x = torch.rand(n, dtype=torch.float64, device="cuda")
for alg in algs:
    tb = float("inf")
    f = None
    for rep in range(3):
        del f
        torch.cuda.synchronize()
        t0 = time.time()
        f = sp.build_format(alg, a, 8)
        torch.cuda.synchronize()
        tb = min(tb, time.time() - t0)
    y = torch.empty(m, dtype=torch.float64, device="cuda")
    for _ in range(5):
        sp.run_spmv(alg, f, x, y, p=8)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps):
        sp.run_spmv(alg, f, x, y, p=8)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    rep = sp.storage_report(f)
    byts = rep.total() + 8 * n + 8 * m
    print(f"{sp.algorithm_name(alg):8s} build {tb*1e3:8.2f} ms  spmv {ms*1e3:8.1f} us  "
          f"{2*v.numel()/ms/1e6:8.1f} GFLOP/s  {byts/ms/1e6:8.1f} GB/s  storage {rep.total()/1e6:.1f} MB",
          flush=True)
    del f
