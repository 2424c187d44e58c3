"""Dev tool: time engines on one BASELINE config under build/run-time env variants (not product).

usage: python tools/engine_time.py CFG ALG[,ALG...] [VARIANT ...]
  VARIANT = "ENV=VAL,ENV=VAL" set for the build and the multiplies of that variant
y of every run is compared with the merge engine's (tolerance 1e-12 * sum |a_ij x_j| is checked
by the tests; here the max relative difference is printed as a sanity check).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402


def time_us(fn, reps=30):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(3):
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps * 1e3)
    return best


cfg = int(sys.argv[1])
algs = [int(a) for a in sys.argv[2].split(",")]
variants = sys.argv[3:] or [""]
name, mk = gen.CONFIGS[cfg]
m, n, r, c, v = mk()
a = sp.TripletMatrix(m, n, r, c, v)
nnz = v.numel()
x = torch.rand(n, dtype=torch.float64, device="cuda")
fm = sp.build_format(2, a, 1)
y_ref = sp.run_spmv(2, fm, x)
scale = sp.run_spmv(2, sp.build_format(2, sp.TripletMatrix(m, n, r, c, v.abs()), 1), x.abs())
del fm
for var in variants:
    env = dict(kv.split("=", 1) for kv in var.split(",") if kv)
    os.environ.update(env)
    for alg in algs:
        f = sp.build_format(alg, a, 16)
        y = torch.empty(m, dtype=torch.float64, device="cuda")
        us = time_us(lambda: sp.run_spmv(alg, f, x, y, p=16))
        sp.run_spmv(alg, f, x, y, p=16)
        err = float(((y - y_ref).abs() / scale.clamp_min(1e-300)).max())
        byts = sp.storage_report(f).total() + 8 * n + 8 * m
        print(f"{name} {sp.algorithm_name(alg):8s} [{var or 'default'}]: {us:8.1f} us  {byts/us/1e3:7.1f} GB/s  "
              f"err/sum|ax| {err:.2e}", flush=True)
        del f
    for k in env:
        os.environ.pop(k)
