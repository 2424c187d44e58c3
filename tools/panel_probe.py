"""Dev probe: does a column-panel split of A help merge-CSR when x exceeds the L2?

For config C (3, 4, 5 or 2), time merge-CSR on the whole matrix, then on K column panels of
equal width (each a CRS of the entries with col in [k*W, (k+1)*W), full column dimension), run
back to back.  The sum of the panel times (plus ~2 y passes per extra panel, reported
separately) against the whole-matrix time says whether panelled gathers pay.

usage: python tools/panel_probe.py CFG [K,K,...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402

MERGE = 2


def time_us(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ks = [int(k) for k in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 4]
name, mk = gen.CONFIGS[cfg]
m, n, r, c, v = mk()
nnz = v.numel()
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.empty(m, dtype=torch.float64, device="cuda")
f = sp.build_format(MERGE, sp.TripletMatrix(m, n, r, c, v), 8)
t_full = time_us(lambda: sp.run_spmv(MERGE, f, x, y, p=8))
y_full = y.clone()
del f
print(f"{name}: nnz={nnz} whole matrix merge {t_full:.1f} us ({2 * nnz / t_full / 1e3:.1f} GFLOP/s)", flush=True)
yp = torch.empty(m, dtype=torch.float64, device="cuda")
t_yadd = time_us(lambda: y.add_(yp))
for k in ks:
    w = (n + k - 1) // k
    pid = (c.to(torch.int64) & 0xFFFFFFFF) // w
    fs = []
    for i in range(k):
        sel = pid == i
        fs.append(sp.build_format(MERGE, sp.TripletMatrix(m, n, r[sel].contiguous(), c[sel].contiguous(),
                                                          v[sel].contiguous()), 8))
        del sel
    ys = [torch.empty(m, dtype=torch.float64, device="cuda") for _ in range(k)]
    each = [time_us(lambda i=i: sp.run_spmv(MERGE, fs[i], x, ys[i], p=8)) for i in range(k)]

    def all_panels():
        for i in range(k):
            sp.run_spmv(MERGE, fs[i], x, ys[i], p=8)
    t_all = time_us(all_panels)
    tot = sum(ys)
    err = (tot - y_full).abs().max().item()
    print(f"  K={k}: panels {' '.join(f'{t:.0f}' for t in each)} us; back to back {t_all:.1f} us "
          f"+ {k - 1} y adds x {t_yadd:.1f} us = {t_all + (k - 1) * t_yadd:.1f} us "
          f"(whole {t_full:.1f}); max |dy| {err:.2e}", flush=True)
    del fs, ys, tot
