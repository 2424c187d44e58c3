"""Dev tool: read-bandwidth and x-gather floors on the cfg2 matrix (not part of the product)."""
import ctypes as C
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402

so = os.path.join(HERE, "libmicrobench.so")
if not os.path.exists(so):
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                    "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "microbench.cu")], check=True)
L = C.CDLL(so)
for f in (L.mb_stream_read, L.mb_gather_x, L.mb_gather_mul):
    f.restype = C.c_int
L.mb_stream_read.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_void_p]
L.mb_gather_x.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
L.mb_gather_mul.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


s = torch.cuda.current_stream().cuda_stream
buf = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
out = torch.zeros(1, dtype=torch.float64, device="cuda")
for blocks in (148 * 4, 148 * 8, 148 * 16, 148 * 32):
    ms = timeit(lambda: L.mb_stream_read(buf.data_ptr(), buf.numel(), out.data_ptr(), blocks, s))
    print(f"stream read 2 GiB blocks={blocks}: {buf.numel() / ms / 1e6:.0f} GB/s", flush=True)
del buf
m, n, r, c, v = gen.rmat_device(22)
f = sp.build_format(2, sp.TripletMatrix(m, n, r, c, v), 1)
col = sp.capi.load()
ptr = C.c_void_p()
nb = C.c_uint64()
col.spmvlab_cuda_format_array(f.handle, b"col_ind", C.byref(ptr), C.byref(nb))
colp = ptr.value
col.spmvlab_cuda_format_array(f.handle, b"data", C.byref(ptr), C.byref(nb))
valp = ptr.value
nnz = v.numel()
x = torch.rand(n, dtype=torch.float64, device="cuda")
for blocks in (148 * 8, 148 * 16):
    ms = timeit(lambda: L.mb_gather_x(colp, nnz, x.data_ptr(), out.data_ptr(), blocks, s))
    print(f"x gather only ({nnz} gathers + 4B col stream) blocks={blocks}: {ms*1e3:.1f} us", flush=True)
    ms = timeit(lambda: L.mb_gather_mul(colp, valp, nnz, x.data_ptr(), out.data_ptr(), blocks, s))
    print(f"gather*val (12B/nnz stream + gather) blocks={blocks}: {ms*1e3:.1f} us  "
          f"{12*nnz/ms/1e6:.0f} GB/s of A", flush=True)
# random permutation of columns (no locality) for comparison
cperm = torch.randint(0, n, (nnz,), device="cuda", dtype=torch.int32)
ms = timeit(lambda: L.mb_gather_x(cperm.data_ptr(), nnz, x.data_ptr(), out.data_ptr(), 148 * 16, s))
print(f"x gather with uniformly random columns: {ms*1e3:.1f} us", flush=True)
L.mb_gather_mul_tiled.restype = C.c_int
L.mb_gather_mul_tiled.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
for th in (128, 256):
    ms = timeit(lambda: L.mb_gather_mul_tiled(colp, valp, nnz, x.data_ptr(), out.data_ptr(), th, s))
    print(f"gather*val tiled one-CTA-per-tile threads={th}: {ms*1e3:.1f} us", flush=True)
L.mb_gather_mul_tiled_meta.restype = C.c_int
L.mb_gather_mul_tiled_meta.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int,
                                       C.c_void_p]
starts = (torch.arange((nnz + 895) // 896, device="cuda", dtype=torch.int64) * 896).to(torch.int32)
for st in (0, 1):
    ms = timeit(lambda: L.mb_gather_mul_tiled_meta(colp, valp, starts.data_ptr(), nnz, x.data_ptr(), out.data_ptr(),
                                                   st, s))
    print(f"gather*val tiled + dependent tile-start load, smem stage={st}: {ms*1e3:.1f} us", flush=True)
L.mb_gather_mul_warp_stage.restype = C.c_int
L.mb_gather_mul_warp_stage.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
ms = timeit(lambda: L.mb_gather_mul_warp_stage(colp, valp, nnz, x.data_ptr(), out.data_ptr(), s))
print(f"gather*val warp-private smem staging (syncwarp): {ms*1e3:.1f} us", flush=True)
L.mb_gather_mul_blocked4.restype = C.c_int
L.mb_gather_mul_blocked4.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                     C.c_void_p]
for q in (1, 2):
    for blocks in (148 * 8, 148 * 16):
        ms = timeit(lambda: L.mb_gather_mul_blocked4(colp, valp, nnz, x.data_ptr(), out.data_ptr(), blocks, q, s))
        print(f"gather*val lane-blocked (4 consecutive per lane, 128/256-bit loads) q={q} blocks={blocks}: "
              f"{ms*1e3:.1f} us", flush=True)
