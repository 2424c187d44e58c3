"""Dev tool: merge-CSR with and without the hot-x plan on one BASELINE config (not product).

usage: python tools/hot_merge_probe.py [CFG] [VARIANT ...]
  VARIANT = "ENV=VAL,ENV=VAL" build-time overrides (SPMVLAB_MERGE_HOT_SLOTS, SPMVLAB_MERGE_HOT_TILES, ...)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402

MERGE = 2


def time_us(fn, reps=50):
    for _ in range(5):
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


cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
variants = sys.argv[2:] or ["SPMVLAB_MERGE_HOT=0", ""]
name, mk = gen.CONFIGS[cfg]
m, n, r, c, v = mk()
a = sp.TripletMatrix(m, n, r, c, v)
nnz = v.numel()
x = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
absA = sp.build_format(MERGE, sp.TripletMatrix(m, n, r, c, v.abs()), 1, opt=None) if False else None
y_ref = None
for var in variants:
    env = dict(kv.split("=", 1) for kv in var.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    torch.cuda.synchronize()
    t0 = time.time()
    f = sp.build_format(MERGE, a, 1)
    torch.cuda.synchronize()
    tb = time.time() - t0
    for k, val in old.items():
        if val is None:
            os.environ.pop(k)
        else:
            os.environ[k] = val
    y = torch.empty(m, dtype=torch.float64, device="cuda")
    us = time_us(lambda: sp.run_spmv(MERGE, f, x, y, p=1))
    sp.run_spmv(MERGE, f, x, y, p=1)
    torch.cuda.synchronize()
    if y_ref is None:
        y_ref = y.clone()
        err = 0.0
    else:
        err = float(((y - y_ref).abs() / (y_ref.abs() + 1e-300)).max())
    byts = sp.storage_report(f).total() + 8 * n + 8 * m
    print(f"{name} [{var or 'default'}]: build {tb*1e3:.1f} ms  spmv {us:.1f} us  {2*nnz/us/1e3:.1f} GFLOP/s  "
          f"{byts/us/1e3:.1f} GB/s  max rel diff vs first {err:.3e}", flush=True)
    del f
