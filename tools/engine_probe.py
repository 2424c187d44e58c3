"""Dev tool: per-engine SpMV timing on a BASELINE config (CUDA events, L2 flushed between reps).
usage: python tools/engine_probe.py CFG [ALGS] [--reps N] [--once] [--p P]
  --once: build each engine and run ONE multiply (for ncu -k captures)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int)
ap.add_argument("algs", nargs="?", default="0,1,2,3,4,5,6,7,8,9,10")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--once", action="store_true")
ap.add_argument("--p", type=int, default=8)
ap.add_argument("--det", action="store_true", help="deterministic builds of the blocked formats")
args = ap.parse_args()
name, fn = gen.CONFIGS[args.cfg]
m, n, r, c, v = fn("cuda")
a = sp.TripletMatrix(m, n, r, c, v)
x = torch.rand(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
y = torch.empty(m, dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
print(f"{name}: m={m} nnz={v.numel()}", flush=True)
for alg in [int(s) for s in args.algs.split(",")]:
    torch.cuda.synchronize()
    t0 = time.time()
    f = sp.build_format(alg, a, args.p, sp.EngineOptions(deterministic=args.det))
    torch.cuda.synchronize()
    tb = time.time() - t0
    if args.once:
        sp.run_spmv(alg, f, x, y, p=args.p)
        torch.cuda.synchronize()
        print(sp.algorithm_name(alg), "done", flush=True)
        del f
        continue
    for _ in range(3):
        sp.run_spmv(alg, f, x, y, p=args.p)
    ts = []
    for _ in range(args.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sp.run_spmv(alg, f, x, y, p=args.p)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    rep = sp.storage_report(f)
    byts = rep.total() + 8 * n + 8 * m
    print(f"{sp.algorithm_name(alg):8s} build {tb*1e3:8.2f} ms  spmv min {ts[0]:8.1f} med {ts[len(ts)//2]:8.1f} us  "
          f"{byts/ts[0]/1e3:7.1f} GB/s  ({2*v.numel()/ts[0]/1e3:6.1f} GFLOP/s)", flush=True)
    del f
    sp.release_cached_memory()
