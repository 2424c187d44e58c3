"""Dev tool: loop time per iteration vs iteration count (cfg2, merge engine)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402

m, n, r, c, v = gen.CONFIGS[2][1]()
f = sp.build_format(2, sp.TripletMatrix(m, n, r, c, v), 1)
x0 = torch.rand(n, dtype=torch.float64, device="cuda")
work = torch.empty_like(x0)
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for fused in ("1", "0"):
    os.environ["SPMVLAB_ITER_FUSED"] = fused
    for normalize, norms in ((True, False), (False, False), (False, True)):
        out = []
        for it in (1, 2, 4, 8, 16, 32, 64):
            x = x0.clone()
            with torch.cuda.stream(s):
                e0.record(s)
                sp.iterate(2, f, x, it, normalize=normalize, norms=norms, work=work, stream=s)
                e1.record(s)
            e1.synchronize()
            out.append(f"{it}:{e0.elapsed_time(e1) / it * 1e3:.0f}")
        print(f"fused={fused} normalize={normalize:d} norms={norms:d}  us/iter " + " ".join(out),
              f" sum={float(x.sum()):.6g}", flush=True)
