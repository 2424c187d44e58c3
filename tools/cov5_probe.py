"""Dev tool: share of each column panel's gathers the hot-x slots would cover at cfg5 (R-MAT s26)."""
import torch, sys
sys.path.insert(0, "/root/repo")
from paper_2502_19284_b200 import gen
m, n, r, c, v = gen.CONFIGS[5][1]()
cc = c.to(torch.int64) & 0xFFFFFFFF
cnt = torch.bincount(cc, minlength=n)
nnz = cc.numel()
del r, v, c
K = 3
w = (n + K - 1) // K
for k in range(K):
    seg = cnt[k * w:(k + 1) * w]
    tot = float(seg.sum())
    for H in (12288, 16384, 24576):
        top = torch.topk(seg, H).values
        print(f"panel {k}: nnz share {tot / nnz:.3f}; top {H} cover {float(top.sum()) / tot:.3f} of the panel (min count {int(top[-1])})", flush=True)
top = torch.topk(cnt, 12288).values
print("whole matrix top 12288 cover", float(top.sum()) / nnz)
