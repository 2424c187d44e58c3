"""Dev tool: shared-memory copy of the hottest x entries vs plain LDG gathers (not product).

usage: python tools/hotx_probe.py [CFG]   (default cfg2)
"""
import ctypes as C
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402

so = os.path.join(HERE, "libhotx_probe.so")
if not os.path.exists(so):
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                    "-Xcompiler", "-fPIC", "-lineinfo", "-o", so, os.path.join(HERE, "hotx_probe.cu")], check=True)
L = C.CDLL(so)
V, U64, U32, I = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
L.hp_cluster.argtypes = [I, I, V, V, U64, V, V, U32, V, V]
L.hp_run.argtypes = [I, I, I, V, V, U64, V, V, U32, V, V]


def timeit(fn, reps=20):
    for _ in range(3):
        rc = fn()
        if rc:
            return None
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
name, mk = gen.CONFIGS[cfg]
m, n, r, c, v = mk()
f = sp.build_format(2, sp.TripletMatrix(m, n, r, c, v), 1)
del r, c, v
col = f.array_device("col_ind")
val = f.array_device("data")
nnz = val.numel()
passes = nnz // 128
x = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.zeros(1, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
cnt = torch.bincount(col.to(torch.int64) & 0xFFFFFFFF, minlength=n)
print(f"{name}: nnz {nnz} passes {passes}", flush=True)
y = torch.empty(m, dtype=torch.float64, device="cuda")
print(f"merge engine: {timeit(lambda: (sp.run_spmv(2, f, x, y, p=1), 0)[1]):.1f} us", flush=True)
res = {}
CONTIG = int(os.environ.get("CONTIG", "0"))

tref = float((val[: passes * 128] * x[col[: passes * 128]]).sum())
print("torch sum", tref, flush=True)
for shape, label in ((0, "8w x6"), (1, "24w x2"), (2, "32w x1"), (3, "16w x3"), (4, "16w x2")):
    col32 = col.to(torch.int32)
    fn = lambda: L.hp_run(1, CONTIG, shape, col32.data_ptr(), val.data_ptr(), passes, x.data_ptr(), x.data_ptr(), 0,  # noqa
                          out.data_ptr(), s)
    out.zero_()
    fn()
    torch.cuda.synchronize()
    ref = out.item()
    print(f"ldg {label}: {timeit(fn):.1f} us sum={ref!r}", flush=True)
for H, shapes in ((2048, (0, 1, 3)), (4096, (0, 1, 3)), (8192, (1, 3, 4)), (12288, (1, 4)), (16384, (2, 4)),
                  (24576, (2,))):
    top = torch.topk(cnt, H).indices
    cover = float(cnt[top].sum()) / nnz
    slot = torch.full((n,), -1, dtype=torch.int64, device="cuda")
    slot[top] = torch.arange(H, device="cuda")
    c64 = col.to(torch.int64) & 0xFFFFFFFF
    sl = slot[c64]
    col2 = torch.where(sl >= 0, (sl | 0x80000000) - (1 << 32), c64).to(torch.int32).contiguous()
    del sl, c64
    xh = x[top].contiguous()
    for shape in shapes:
        fn = lambda: L.hp_run(1, CONTIG, shape, col2.data_ptr(), val.data_ptr(), passes, x.data_ptr(), xh.data_ptr(), H,  # noqa
                              out.data_ptr(), s)
        out.zero_()
        rc = fn()
        torch.cuda.synchronize()
        ok = (abs(out.item() - tref) <= 1e-9 * abs(tref), out.item())
        print(f"hot H={H} ({H*8//1024} KB, {cover:.3f} of gathers) shape {shape}: rc={rc} {timeit(fn):.1f} us ok={ok}",
              flush=True)
    del col2

# cluster-shared hot copies (distributed shared memory): CL CTAs x (H / CL) slots each
for H, CL in ((12288, 1), (24576, 2), (49152, 4), (12288, 2), (24576, 4)):
    top = torch.topk(cnt, H).indices
    cover = float(cnt[top].sum()) / nnz
    slot = torch.full((n,), -1, dtype=torch.int64, device="cuda")
    slot[top] = torch.arange(H, device="cuda")
    c64 = col.to(torch.int64) & 0xFFFFFFFF
    sl = slot[c64]
    col2 = torch.where(sl >= 0, (sl | 0x80000000) - (1 << 32), c64).to(torch.int32).contiguous()
    del sl, c64
    xh = x[top].contiguous()
    fn = lambda: L.hp_cluster(CL, CONTIG, col2.data_ptr(), val.data_ptr(), passes, x.data_ptr(), xh.data_ptr(), H,  # noqa
                              out.data_ptr(), s)
    out.zero_()
    rc = fn()
    torch.cuda.synchronize()
    ok = abs(out.item() - tref) <= 1e-9 * abs(tref)
    print(f"cluster CL={CL} H={H} ({H*8//1024//CL} KB/CTA, {cover:.3f} of gathers): rc={rc} {timeit(fn):.1f} us ok={ok}",
          flush=True)
