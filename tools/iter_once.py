"""Dev tool (ncu target): one plain merge multiply, then 2 loop iterations with rescale and norms."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402

name, fn = gen.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
m, n, r, c, v = fn("cuda")
f = sp.build_format(2, sp.TripletMatrix(m, n, r, c, v), 1)
del r, c, v
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = sp.run_spmv(2, f, x)
sp.iterate(2, f, x, 2, normalize=True)
torch.cuda.synchronize()
print("ok")
