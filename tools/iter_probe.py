"""Dev tool: the application loop's cost over the plain multiply (fused vs separate-pass norms).
usage: python tools/iter_probe.py CFG [ITERS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402

cfg = int(sys.argv[1])
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
name, fn = gen.CONFIGS[cfg]
m, n, r, c, v = fn("cuda")
f = sp.build_format(2, sp.TripletMatrix(m, n, r, c, v), 1)
del r, c, v
sp.release_cached_memory()
x0 = torch.rand(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
y = torch.empty_like(x0)
work = torch.empty_like(x0)
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t_spmv():
    with torch.cuda.stream(s):
        for _ in range(3):
            sp.run_spmv(2, f, x0, y, stream=s)
        e0.record(s)
        for _ in range(iters):
            sp.run_spmv(2, f, x0, y, stream=s)
        e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / iters


def t_iter(normalize, norms, graph):
    x = x0.clone()
    sp.iterate(2, f, x, 2, normalize=normalize, norms=norms, graph=graph, work=work, stream=s)
    s.synchronize()
    e0.record(s)
    sp.iterate(2, f, x, iters, normalize=normalize, norms=norms, graph=graph, work=work, stream=s)
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / iters


base = t_spmv()
print(f"{name}: spmv {base*1e3:.1f} us  panels {f.info['merge_panels']}", flush=True)
for unf in (False, True):
    if unf:
        os.environ["SPMVLAB_ITER_FUSED"] = "0"
    for normalize, norms in ((False, False), (False, True), (True, False), (True, True)):
        for graph in (False, True):
            t = t_iter(normalize, norms, graph)
            print(f"  {'unfused' if unf else 'fused  '} normalize={normalize:d} norms={norms:d} graph={graph:d}: "
                  f"{t*1e3:8.1f} us/iter  ({t/base:.3f}x spmv)", flush=True)
    os.environ.pop("SPMVLAB_ITER_FUSED", None)
