"""Profiling probe (dev tool): build the given engines on R-MAT scale S and run each SpMV once,
so an ncu capture sees exactly one multiply launch per engine.
usage: python tools/probe_blocked.py 22 3,9"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
algs = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [3, 9]
m, n, r, c, v = gen.rmat_device(scale)
a = sp.TripletMatrix(m, n, r, c, v)
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.empty(m, dtype=torch.float64, device="cuda")
for alg in algs:
    f = sp.build_format(alg, a, 8)
    torch.cuda.synchronize()
    sp.run_spmv(alg, f, x, y, p=8)
    torch.cuda.synchronize()
    print(sp.algorithm_name(alg), "items", f.info.get("work_items"), flush=True)
    del f
