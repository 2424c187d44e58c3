"""Dev tool: TMA gather4 / bulk copies vs LDG for merge-CSR's x gathers on the cfg2 matrix (not product)."""
import ctypes as C
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402

so = os.path.join(HERE, "libgather4_probe.so")
if not os.path.exists(so):
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                    "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "gather4_probe.cu")], check=True)
L = C.CDLL(so)
V, U64, I = C.c_void_p, C.c_uint64, C.c_int
L.gp_ldg.argtypes = [V, V, U64, V, V, I, V]
L.gp_gather4.argtypes = [V, V, U64, V, U64, V, I, I, I, I, I, I, V]
L.gp_bulk16.argtypes = [V, V, U64, V, V, I, I, I, V]


def timeit(fn, reps=20):
    for _ in range(3):
        rc = fn()
        if rc:
            return None, rc
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3, 0


s = torch.cuda.current_stream().cuda_stream
scale = int(os.environ.get("SCALE", "22"))
m, n, r, c, v = gen.rmat_device(scale)
f = sp.build_format(2, sp.TripletMatrix(m, n, r, c, v), 1)
lib = sp.capi.load()
ptr, nb = C.c_void_p(), C.c_uint64()
lib.spmvlab_cuda_format_array(f.handle, b"col_ind", C.byref(ptr), C.byref(nb))
colp = ptr.value
lib.spmvlab_cuda_format_array(f.handle, b"data", C.byref(ptr), C.byref(nb))
valp = ptr.value
nnz = v.numel()
passes = nnz // 128
x = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.zeros(1, dtype=torch.float64, device="cuda")
print(f"scale {scale}: nnz {nnz}, passes {passes} ({passes*128} elements timed)", flush=True)


def check(fn):
    out.zero_()
    rc = fn()
    torch.cuda.synchronize()
    return rc, out.item()


ref = None
for blocks in (148 * 4, 148 * 6, 148 * 8, 148 * 16):
    fn = lambda: L.gp_ldg(colp, valp, passes, x.data_ptr(), out.data_ptr(), blocks, s)  # noqa: E731
    rc, val = check(fn)
    ref = val
    us, _ = timeit(fn)
    print(f"ldg blocks={blocks}: {us:.1f} us  sum={val:.12e}", flush=True)

L.gp_hyb.argtypes = [V, V, U64, V, U64, V, I, I, I, I, I, V]
for S, W in ((2, 8), (3, 8)):
    for occ in (2, 3):
        blocks = 148 * occ
        fn = lambda: L.gp_gather4(colp, valp, passes, x.data_ptr(), n, out.data_ptr(), blocks, 4, S, W, 1, 0, s)  # noqa
        rc, val = check(fn)
        if rc:
            continue
        us, _ = timeit(fn)
        print(f"gather4 R=4 S={S} W={W} blocks={blocks}: {us:.1f} us ok={abs(val - ref) <= 1e-9 * abs(ref)}",
              flush=True)
for kind, cfgs in ((0, ((2, 8, 2), (2, 8, 3), (2, 8, 4), (3, 8, 3), (2, 4, 3), (2, 8, 6))),
                   (1, ((2, 8, 8), (2, 8, 12), (2, 8, 16), (3, 8, 12), (4, 8, 8), (4, 8, 12), (2, 4, 12)))):
    for S, W, K in cfgs:
        for occ in (2, 3, 4, 6, 8):
            smem = W * S * (32 if kind == 0 else K) * 128
            if smem * occ > 220 * 1024 or W * 32 * occ > 2048:
                continue
            blocks = 148 * occ
            fn = lambda: L.gp_hyb(colp, valp, passes, x.data_ptr(), n, out.data_ptr(), blocks, kind, S, W, K, s)  # noqa
            rc, val = check(fn)
            if rc:
                print(f"hyb kind={kind} S={S} W={W} K={K}: rc {rc}", flush=True)
                break
            us, _ = timeit(fn)
            name = "pass 1/K via TMA" if kind == 0 else "lanes<K via TMA"
            print(f"hyb[{name}] S={S} W={W} K={K} blocks={blocks}: {us:.1f} us "
                  f"ok={abs(val - ref) <= 1e-9 * abs(ref)}", flush=True)

for S, W in ((4, 4), (8, 4), (4, 8), (8, 8)):
    for occ in (2, 4, 8):
        smem = W * S * 128 * 16
        if smem * occ > 220 * 1024 or W * 32 * occ > 2048:
            continue
        blocks = 148 * occ
        fn = lambda: L.gp_bulk16(colp, valp, passes, x.data_ptr(), out.data_ptr(), blocks, S, W, s)  # noqa: E731
        rc, val = check(fn)
        if rc:
            print(f"bulk16 S={S} W={W}: rc {rc}", flush=True)
            continue
        us, _ = timeit(fn)
        print(f"bulk16 S={S} W={W} blocks={blocks}: {us:.1f} us ok={abs(val - ref) <= 1e-9 * abs(ref)}", flush=True)
