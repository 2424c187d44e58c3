"""Dev tool: distribution of COO->format build times (10 builds per engine) on R-MAT scale S."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_19284_b200 as sp
from paper_2502_19284_b200 import gen
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
algs = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2]
m, n, r, c, v = gen.rmat_device(scale)
a = sp.TripletMatrix(m, n, r, c, v)
for alg in algs:
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f = sp.build_format(alg, a, 8)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
        del f
    print(sp.algorithm_name(alg), " ".join(f"{t:.1f}" for t in ts), flush=True)
