"""Dev tool: a few loop iterations on cfg2 (for an ncu launch list)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402

m, n, r, c, v = gen.CONFIGS[2][1]()
f = sp.build_format(2, sp.TripletMatrix(m, n, r, c, v), 1)
x = torch.rand(n, dtype=torch.float64, device="cuda")
normalize = int(sys.argv[1]) if len(sys.argv) > 1 else 1
norms = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sp.iterate(2, f, x, 6, normalize=bool(normalize), norms=bool(norms))
torch.cuda.synchronize()
print("done", x[:4].tolist())
