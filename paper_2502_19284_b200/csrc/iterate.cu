// iterate.cu -- the iterated multiply x_{k+1} = A x_k of the cfg5 application (SURVEY.md §8e and
// §8f item 2) on one device.
//
// The reference has no loop of its own: BASELINE cfg5 is "x <- A x for 100 iterations" around
// run_spmv (inc/engine.hpp:126-148).  Iteration k produces y = A x_k, the convergence norms
// residual_k = ||A x_k - x_k||_1 and mass_k = sum(A x_k) -- with a unit-mass x_k, 1 - mass_k is the
// leakage through empty columns of the column-normalised matrix -- and optionally rescales
// x_{k+1} = y / mass_k to unit mass (without rescaling residual_k = ||x_{k+1} - x_k||_1).
//
//  * Merge engine (the north-star engine): the norms are FUSED into the multiply.  The merge tile
//    kernel and its carry fix-up add each row's final value into per-tile / per-warp (mass,
//    residual) partial sums as the row is stored (one extra row-indexed read of x_k[r]), and a
//    small reduction kernel (norms_finish_kernel) combines the partials in a fixed order.  The
//    rescale is deferred: the stored vector is u_{k+1} = A x_k and x_{k+1} = u_{k+1} / mass_k, so
//    iteration k + 1 multiplies u_{k+1} and scales every value it stores by 1 / mass_k (kept in
//    device memory); the final iterate is rescaled once at the end.  No pass over the vectors
//    besides the multiply itself.
//  * Other engines: the multiply, then one pass over (x_k, y) for (mass, residual) and, with
//    rescaling, one pass scaling y.
// Reductions are deterministic: fixed per-CTA grid-stride partial sums, the last CTA to finish
// (ticket counter) reduces the partials in a fixed tree order.
//
// Where the norms of iteration k go is decided on the device (an iteration counter in the scratch
// block), so the launch parameters of every iteration pair (x -> work -> x) are identical: graph
// mode captures ONE pair and replays it iters / 2 times.
#include <algorithm>
#include <string>
#include <utility>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {
extern thread_local std::string g_last_error;
namespace {

constexpr int kRedThreads = 256;
constexpr unsigned kRedBlocks = 8 * kNumSMs;
constexpr int kRedUnroll = 4;

struct IterScratch {
  double partial[2 * kRedBlocks];
  double pair[2];     // (residual, mass) of the current iteration when the caller keeps no norms
  double inv_scale;   // fused path: x_k = stored vector * inv_scale (deferred normalisation)
  unsigned ticket;    // CTAs finished in the current reduction
  unsigned iter;      // iteration index (selects norms + 2 * iter)
};

__device__ __forceinline__ double* iter_out(IterScratch* sc, double* norms) {
  return norms ? norms + 2ull * sc->iter : sc->pair;
}

// MODE bit 0: accumulate the mass of y; bit 1: scale y by 1 / (mass of this iteration) first;
// bit 2: accumulate |y - x|.  Writes out[0] = diff, out[1] = mass (those accumulated); with
// bit 3 (last reduction of the iteration) the iteration counter advances.
template <int MODE>
__global__ void __launch_bounds__(kRedThreads) iter_reduce_kernel(const double* __restrict__ x,
                                                                  double* __restrict__ y, uint64_t n,
                                                                  IterScratch* sc, double* norms) {
  double scale = 1.0;
  if (MODE & 2) scale = 1.0 / iter_out(sc, norms)[1];
  double d = 0.0, s = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (kRedUnroll - 1) * stride < n; i += kRedUnroll * stride) {
    double v[kRedUnroll], xv[kRedUnroll];
#pragma unroll
    for (int u = 0; u < kRedUnroll; ++u) {
      v[u] = y[i + u * stride];
      if (MODE & 4) xv[u] = x[i + u * stride];
    }
#pragma unroll
    for (int u = 0; u < kRedUnroll; ++u) {
      if (MODE & 2) {
        v[u] *= scale;
        y[i + u * stride] = v[u];
      }
      if (MODE & 1) s += v[u];
      if (MODE & 4) d += fabs(v[u] - xv[u]);
    }
  }
  for (; i < n; i += stride) {
    double v = y[i];
    if (MODE & 2) {
      v *= scale;
      y[i] = v;
    }
    if (MODE & 1) s += v;
    if (MODE & 4) d += fabs(v - x[i]);
  }
  __shared__ double sd[kRedThreads / 32], ss[kRedThreads / 32];
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
      ss[warp] = b;
    }
    __syncthreads();
    a = 0.0;
    b = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) {
      a += sd[w];
      b += ss[w];
    }
  };
  block_sum(d, s);
  if (threadIdx.x == 0) {
    sc->partial[2 * blockIdx.x] = d;
    sc->partial[2 * blockIdx.x + 1] = s;
    __threadfence();
    last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double td = 0.0, ts = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    td += __ldcg(sc->partial + 2 * b);
    ts += __ldcg(sc->partial + 2 * b + 1);
  }
  __syncthreads();  // sd / ss reuse
  block_sum(td, ts);
  if (threadIdx.x == 0) {
    double* out = iter_out(sc, norms);
    if (MODE & 4) out[0] = td;
    if (MODE & 1) out[1] = ts;
    sc->ticket = 0;  // ready for the next reduction (stream order)
    if (MODE & 8) sc->iter += 1;
  }
}

// Fused norms: the (mass, residual) partials the merge multiply left per tile and per fix-up warp,
// reduced in a fixed order (grid-stride per thread, CTA tree, last CTA over the CTA sums).  Writes
// out[0] = residual, out[1] = mass; with `normalize` the next iteration's deferred scale
// inv_scale = 1 / mass; advances the iteration counter.
__global__ void __launch_bounds__(kRedThreads) norms_finish_kernel(const double* __restrict__ tile_part,
                                                                   uint64_t ntile, const double* __restrict__ fix_part,
                                                                   uint64_t nfix, IterScratch* sc, double* norms,
                                                                   int normalize) {
  double res = 0.0, mass = 0.0;
  const uint64_t total = ntile + nfix;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const double* p = i < ntile ? tile_part + 2 * i : fix_part + 2 * (i - ntile);
    mass += p[0];
    res += p[1];
  }
  __shared__ double sd[kRedThreads / 32], ss[kRedThreads / 32];
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
      ss[warp] = b;
    }
    __syncthreads();
    a = 0.0;
    b = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) {
      a += sd[w];
      b += ss[w];
    }
  };
  block_sum(res, mass);
  if (threadIdx.x == 0) {
    sc->partial[2 * blockIdx.x] = res;
    sc->partial[2 * blockIdx.x + 1] = mass;
    __threadfence();
    last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double tr = 0.0, tm = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    tr += __ldcg(sc->partial + 2 * b);
    tm += __ldcg(sc->partial + 2 * b + 1);
  }
  __syncthreads();
  block_sum(tr, tm);
  if (threadIdx.x == 0) {
    double* out = iter_out(sc, norms);
    out[0] = tr;
    out[1] = tm;
    if (normalize) sc->inv_scale = 1.0 / tm;
    sc->ticket = 0;
    sc->iter += 1;
  }
}

// y = x * inv_scale (the fused path's final rescale; in place when y == x)
__global__ void scale_kernel(const double* x, double* y, uint64_t n, const IterScratch* sc) {
  const double s = sc->inv_scale;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    y[i] = x[i] * s;
}

__global__ void init_scratch_kernel(IterScratch* sc) {
  sc->inv_scale = 1.0;
  sc->ticket = 0;
  sc->iter = 0;
}

// Partial-sum buffers of the fused path, sized from the last panel's tile count.
struct FusedNorms {
  double* tile_part = nullptr;
  double* fix_part = nullptr;
  uint64_t ntile = 0, nfix = 0;
};

int one_iteration_fused(const Format& f, const double* cur, double* nxt, bool normalize, double* norms,
                        IterScratch* sc, const FusedNorms& fb, cudaStream_t s) {
  NormCtx nc;
  nc.xr = cur;
  nc.inv_scale = normalize ? &sc->inv_scale : nullptr;
  nc.tile_part = fb.tile_part;
  nc.fix_part = fb.fix_part;
  if (int rc = spmv_merge(f, cur, nxt, s, nullptr, &nc)) return rc;
  const uint64_t want = (fb.ntile + fb.nfix + kRedThreads * 8 - 1) / (kRedThreads * 8);
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(kRedBlocks, want));
  norms_finish_kernel<<<grid, kRedThreads, 0, s>>>(fb.tile_part, fb.ntile, fb.fix_part, fb.nfix, sc, norms,
                                                    normalize ? 1 : 0);
  note_launch();
  return kOk;
}

template <int MODE>
void launch_reduce(const double* x, double* y, uint64_t n, IterScratch* sc, double* norms, cudaStream_t s) {
  const uint64_t want = (n + (uint64_t)kRedThreads * kRedUnroll - 1) / ((uint64_t)kRedThreads * kRedUnroll);
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(kRedBlocks, want));
  iter_reduce_kernel<MODE><<<grid, kRedThreads, 0, s>>>(x, y, n, sc, norms);
  note_launch();
}

int one_iteration(const SpmvFn& multiply, const double* cur, double* nxt, uint64_t n, bool normalize, double* norms,
                  IterScratch* sc, cudaStream_t s) {
  if (int rc = multiply(cur, nxt, s)) return rc;
  if (normalize) {
    launch_reduce<1 | 4>(cur, nxt, n, sc, norms, s);  // mass of A x_k and |A x_k - x_k|
    launch_reduce<2 | 8>(cur, nxt, n, sc, norms, s);  // rescale to unit mass
  } else if (norms) {
    launch_reduce<1 | 4 | 8>(cur, nxt, n, sc, norms, s);
  }
  return kOk;
}

}  // namespace

int iterate(const Format& f, const SpmvFn& multiply, double* x, double* work, uint32_t iters, int flags,
            double* norms, cudaStream_t s, bool fused_merge) {
  const uint64_t n = f.n;
  const bool normalize = flags & 1, graph = flags & 2;
  // the fused path needs no norms pass at all; without norms or rescaling there is nothing to fuse
  const bool fused = fused_merge && f.merge_tiles > 0 && (normalize || norms);
  IterScratch* sc = nullptr;
  if (cudaMallocAsync(&sc, sizeof(IterScratch), s) != cudaSuccess) {
    cudaGetLastError();
    g_last_error = "device allocation failed (iterate scratch)";
    return kNoMemory;
  }
  cudaMemsetAsync(sc, 0, sizeof(IterScratch), s);
  init_scratch_kernel<<<1, 1, 0, s>>>(sc);
  FusedNorms fb;
  if (fused) {
    const uint32_t kl = f.merge_panels - 1;
    fb.ntile = f.panel_tile_off[kl + 1] - f.panel_tile_off[kl];
    fb.nfix = (fb.ntile + 31) / 32;
    if (cudaMallocAsync(&fb.tile_part, 16 * (fb.ntile + fb.nfix + 1), s) != cudaSuccess) {
      cudaGetLastError();
      cudaFreeAsync(sc, s);
      g_last_error = "device allocation failed (fused norm partials)";
      return kNoMemory;
    }
    fb.fix_part = fb.tile_part + 2 * fb.ntile;
  }
  auto step = [&](const double* cur, double* nxt) {
    return fused ? one_iteration_fused(f, cur, nxt, normalize, norms, sc, fb, s)
                 : one_iteration(multiply, cur, nxt, n, normalize, norms, sc, s);
  };
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
      rc = step(x, work);
      if (rc == kOk) rc = step(work, x);
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
  for (; rc == kOk && done < iters; ++done) {
    rc = step(cur, nxt);
    std::swap(cur, nxt);
  }
  if (rc == kOk && fused && normalize && n) {  // the deferred rescale of the last iterate
    scale_kernel<<<grid_for(n, 256), 256, 0, s>>>(cur, x, n, sc);
    note_launch();
  } else if (rc == kOk && cur != x && n) {
    cudaMemcpyAsync(x, cur, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
  }
  if (fb.tile_part) cudaFreeAsync(fb.tile_part, s);
  cudaFreeAsync(sc, s);
  return rc ? rc : check_launch("iterate");
}

}  // namespace spmvcu
