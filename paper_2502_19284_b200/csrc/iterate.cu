// iterate.cu -- the iterated multiply x_{k+1} = A x_k of the cfg5 application (SURVEY.md §8e and
// §8f item 2) on one device.
//
// The reference has no loop of its own: BASELINE cfg5 is "x <- A x for 100 iterations" around
// run_spmv (inc/engine.hpp:126-148).  Iteration k produces y = A x_k, the convergence norms
// residual_k = ||A x_k - x_k||_1 and mass_k = sum(A x_k) -- with a unit-mass x_k, 1 - mass_k is the
// leakage through empty columns of the column-normalised matrix -- and optionally rescales
// x_{k+1} = A x_k / mass_k to unit mass (without rescaling residual_k = ||x_{k+1} - x_k||_1).
//
// One pass per iteration after the multiply, with a deferred scale: the stored vector u_k and a
// device scalar s_k with x_k = s_k u_k.  The engine multiplies the stored vector, y = A u_k, and
// the pass reads y (and u_k for the residual) once: t = s_k y_r = (A x_k)_r is summed into the
// mass and |t - s_k u_k[r]| into the residual; rescaling keeps y as the stored vector and sets
// s_{k+1} = s_k / mass_k (y is written back scaled only when s drifts out of [2^-256, 2^256]).  The
// last iterate is scaled once at the end.  Traffic per row: 16 B with the residual, 8 B for the mass
// alone (the write-back of every rescaled iterate was 24 B; two passes -- mass, then rescale --
// were 32 B and two launches); nothing at all when neither norms nor rescaling are asked for.
//
// Folding the mass and the scale into the merge kernel itself (tile partial sums of the products,
// every stored row scaled) measured SLOWER than this pass: the latency-bound merge kernel loses an
// occupancy step or spills with the extra registers (cfg2 loop 1.15 vs 1.12 x the multiply, cfg5
// 1.14 vs 1.11; per-row residuals in-kernel 1.25-1.29 x).
//
// Reductions are deterministic: fixed per-CTA grid-stride partial sums, the last CTA to finish
// (ticket counter) reduces the partials in a fixed tree order.  Where the norms of iteration k go
// is decided on the device (an iteration counter in the scratch block), so the launch parameters of
// every iteration pair (x -> work -> x) are identical: graph mode captures ONE pair and replays it
// iters / 2 times.
#include <algorithm>
#include <cstdlib>
#include <string>
#include <utility>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {
extern thread_local std::string g_last_error;
namespace {

constexpr int kRedThreads = 256;
constexpr int kRedUnroll = 4;  // double2 per thread per step

__device__ __forceinline__ double* iter_out(IterScratch* sc, double* norms) {
  return norms ? norms + 2ull * sc->iter : sc->pair;
}

__global__ void init_scratch_kernel(IterScratch* sc) {
  sc->scale = 1.0;
  sc->pscale = 1.0;
  sc->ticket = 0;
  sc->iter = 0;
}

// The pass after iteration k's multiply (see the file comment).  RESIDUAL: read u_k and accumulate
// |t - s_k u_k|.  Always: the mass.  RESCALE: x_{k+1} = A x_k / mass_k = (s_k / mass_k) y, so the
// stored vector stays y and only the scalar changes, s_{k+1} = s_k / mass_k -- unless s_k has
// drifted outside [2^-256, 2^256] (y itself then grows or shrinks with every iteration): then t is
// written back and s_{k+1} = 1 / mass_k.  The test is uniform over the grid.
template <bool RESCALE, bool RESIDUAL>
__global__ void __launch_bounds__(kRedThreads) iter_pass_kernel(const double* __restrict__ u, double* __restrict__ y,
                                                                uint64_t n, IterScratch* sc, double* norms) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // launched behind the multiply (PDL)
  const double s = sc->scale;
  const bool write_back = RESCALE && !(fabs(s) >= 0x1p-256 && fabs(s) <= 0x1p256);
  double d = 0.0, m = 0.0;
  const uint64_t n2 = n / 2;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  double2* y2 = reinterpret_cast<double2*>(y);
  const double2* u2 = reinterpret_cast<const double2*>(u);
  const bool vec = ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(u)) & 15u) == 0;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  auto one = [&](double yv, double uv) -> double {
    const double t = s * yv;
    m += t;
    if (RESIDUAL) d += fabs(t - s * uv);
    return t;
  };
  if (vec) {
    for (; i + (kRedUnroll - 1) * stride < n2; i += kRedUnroll * stride) {
      double2 yv[kRedUnroll], uv[kRedUnroll];
#pragma unroll
      for (int k = 0; k < kRedUnroll; ++k) {
        yv[k] = y2[i + k * stride];
        if (RESIDUAL) uv[k] = __ldg(u2 + i + k * stride);
      }
#pragma unroll
      for (int k = 0; k < kRedUnroll; ++k) {
        double2 t;
        t.x = one(yv[k].x, RESIDUAL ? uv[k].x : 0.0);
        t.y = one(yv[k].y, RESIDUAL ? uv[k].y : 0.0);
        if (write_back) y2[i + k * stride] = t;
      }
    }
    for (; i < n2; i += stride) {
      const double2 yv = y2[i];
      const double2 uv = RESIDUAL ? __ldg(u2 + i) : make_double2(0.0, 0.0);
      double2 t;
      t.x = one(yv.x, uv.x);
      t.y = one(yv.y, uv.y);
      if (write_back) y2[i] = t;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) {  // the odd tail element
      const double t = one(y[n - 1], RESIDUAL ? u[n - 1] : 0.0);
      if (write_back) y[n - 1] = t;
    }
  } else {
    for (; i < n; i += stride) {
      const double t = one(y[i], RESIDUAL ? u[i] : 0.0);
      if (write_back) y[i] = t;
    }
  }
  __shared__ double sd[kRedThreads / 32], sm[kRedThreads / 32];
  __shared__ bool last;
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  auto block_sum = [&](double& a, double& b) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_xor_sync(0xFFFFFFFFu, a, off);
      b += __shfl_xor_sync(0xFFFFFFFFu, b, off);
    }
    if (lane == 0) {
      sd[warp] = a;
      sm[warp] = b;
    }
    __syncthreads();
    a = 0.0;
    b = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) {
      a += sd[w];
      b += sm[w];
    }
  };
  block_sum(d, m);
  if (threadIdx.x == 0) {
    sc->partial[2 * blockIdx.x] = d;
    sc->partial[2 * blockIdx.x + 1] = m;
    __threadfence();
    last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double td = 0.0, tm = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    td += __ldcg(sc->partial + 2 * b);
    tm += __ldcg(sc->partial + 2 * b + 1);
  }
  __syncthreads();  // sd / sm reuse
  block_sum(td, tm);
  if (threadIdx.x == 0) {
    double* out = iter_out(sc, norms);
    out[0] = RESIDUAL ? td : 0.0;
    out[1] = tm;
    if (RESCALE) sc->scale = write_back ? 1.0 / tm : s / tm;
    sc->ticket = 0;  // ready for the next reduction (stream order)
    sc->iter += 1;
  }
}

// y = x * scale (the last iterate, once at the end; in place when y == x)
__global__ void scale_kernel(const double* x, double* y, uint64_t n, const IterScratch* sc) {
  const double s = sc->scale;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    y[i] = x[i] * s;
}

template <bool RESCALE, bool RESIDUAL>
void launch_pass(const double* u, double* y, uint64_t n, IterScratch* sc, double* norms, cudaStream_t s) {
  const uint64_t want = (n + 2ull * kRedThreads * kRedUnroll - 1) / (2ull * kRedThreads * kRedUnroll);
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(kRedBlocks, want));
  // programmatic dependent launch: the pass is resident while the multiply's fix-up drains
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kRedThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, iter_pass_kernel<RESCALE, RESIDUAL>, u, y, n, sc, norms);
  note_launch();
}

int one_iteration(const Format& f, const SpmvFn& multiply, bool fused, const double* cur, double* nxt, uint64_t n,
                  bool normalize, double* norms, IterScratch* sc, cudaStream_t s) {
  // (the residual inside the multiply -- NORMS = 2 -- measured slower than this pass: cfg2 346 vs
  // 302 us per iteration; the mass alone is free there: 280 vs 298 us)
  if (fused && normalize && !norms) return spmv_merge_norms(f, cur, nxt, s, sc);
  if (int rc = multiply(cur, nxt, s)) return rc;
  if (normalize && norms) launch_pass<true, true>(cur, nxt, n, sc, norms, s);
  else if (normalize) launch_pass<true, false>(cur, nxt, n, sc, norms, s);
  else if (norms) launch_pass<false, true>(cur, nxt, n, sc, norms, s);
  return kOk;
}

}  // namespace

int iterate(const Format& f, const SpmvFn& multiply, double* x, double* work, uint32_t iters, int flags,
            double* norms, cudaStream_t s, bool merge_engine) {
  const uint64_t n = f.n;
  const bool normalize = flags & 1, graph = flags & 2;
  // norms inside the multiply (hot-x plan of the merge engine); SPMVLAB_ITER_FUSED=0 (developer)
  // keeps the separate pass
  bool fused = merge_engine && merge_norms_supported(f);
  if (const char* e = getenv("SPMVLAB_ITER_FUSED")) fused = fused && atoi(e) != 0;
  IterScratch* sc = nullptr;
  if (cudaMallocAsync(&sc, sizeof(IterScratch), s) != cudaSuccess) {
    cudaGetLastError();
    g_last_error = "device allocation failed (iterate scratch)";
    return kNoMemory;
  }
  cudaMemsetAsync(sc, 0, sizeof(IterScratch), s);
  init_scratch_kernel<<<1, 1, 0, s>>>(sc);
  note_launch();
  int rc = kOk;
  uint32_t done = 0;
  if (graph && iters >= 2) {
    // capture one (x -> work -> x) pair and replay it; the suspended instrumentation brackets and
    // the per-stream scratch were settled by the caller
    cudaGraph_t g = nullptr;
    const uint64_t l0 = spmvlab_cuda_launch_count();
    if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      rc = check_launch("iterate(capture)");
    } else {
      rc = one_iteration(f, multiply, fused, x, work, n, normalize, norms, sc, s);
      if (rc == kOk) rc = one_iteration(f, multiply, fused, work, x, n, normalize, norms, sc, s);
      const cudaError_t ce = cudaStreamEndCapture(s, &g);
      if (rc == kOk && ce != cudaSuccess) rc = check_launch("iterate(capture)");
    }
    cudaGraphExec_t ge = nullptr;
    if (rc == kOk && cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) rc = check_launch("iterate(instantiate)");
    const uint64_t per_pair = spmvlab_cuda_launch_count() - l0;  // kernels in one captured pair
    for (; rc == kOk && done + 2 <= iters; done += 2) {
      if (cudaGraphLaunch(ge, s) != cudaSuccess) rc = check_launch("iterate(launch)");
      if (done) note_launch((unsigned)per_pair);  // the capture counted the first replay
    }
    if (ge) cudaGraphExecDestroy(ge);  // freed once in-flight launches complete
    if (g) cudaGraphDestroy(g);
  }
  double* cur = x;
  double* nxt = work;
  if (done & 1) std::swap(cur, nxt);
  for (; rc == kOk && done < iters; ++done) {
    rc = one_iteration(f, multiply, fused, cur, nxt, n, normalize, norms, sc, s);
    std::swap(cur, nxt);
  }
  if (rc == kOk && normalize && n) {  // x = s * stored vector (in place or into x)
    scale_kernel<<<grid_for(n, 256), 256, 0, s>>>(cur, x, n, sc);
    note_launch();
  } else if (rc == kOk && cur != x && n) {
    cudaMemcpyAsync(x, cur, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
  }
  cudaFreeAsync(sc, s);
  return rc ? rc : check_launch("iterate");
}

}  // namespace spmvcu
