// iterate.cu -- the iterated multiply x_{k+1} = A x_k of the cfg5 application (SURVEY.md §8e and
// §8f item 2) on one device.
//
// The reference has no loop of its own: BASELINE cfg5 is "x <- A x for 100 iterations" around
// run_spmv (inc/engine.hpp:126-148).  Each iteration here is the engine's multiply into the other
// buffer followed by one fused pass over the pair (x_k, x_{k+1}) that produces the convergence
// norms ||x_{k+1} - x_k||_1 and the mass sum(x_{k+1}) -- the mass lost since the previous step is
// the leakage through empty columns of the column-normalised matrix -- and optionally rescales
// x_{k+1} to unit mass.  Reductions are deterministic: fixed per-CTA grid-stride partial sums, the
// last CTA to finish (ticket counter) adds the partials in CTA order.  The loop can be captured
// into one CUDA graph (no per-iteration launch latency for small matrices).
#include <algorithm>
#include <string>
#include <utility>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {
extern thread_local std::string g_last_error;
namespace {

constexpr int kRedThreads = 256;
constexpr unsigned kRedBlocks = 2 * kNumSMs;

// mode bit 0: accumulate the mass of y; bit 1: scale y by 1 / *mass_in first; bit 2: accumulate
// |y - x|.  out[0] = diff, out[1] = mass (only the accumulated ones are written).
template <int MODE>
__global__ void __launch_bounds__(kRedThreads) iter_reduce_kernel(const double* __restrict__ x, double* __restrict__ y,
                                                                  uint64_t n, const double* __restrict__ mass_in,
                                                                  double* __restrict__ partial,
                                                                  unsigned* __restrict__ ticket, double* __restrict__ out) {
  const double scale = (MODE & 2) ? 1.0 / *mass_in : 1.0;
  double d = 0.0, s = 0.0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
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
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    d += __shfl_xor_sync(0xFFFFFFFFu, d, off);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, off);
  }
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sd[warp] = d;
    ss[warp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bd = 0.0, bs = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) {
      bd += sd[w];
      bs += ss[w];
    }
    partial[2 * blockIdx.x] = bd;
    partial[2 * blockIdx.x + 1] = bs;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double td = 0.0, ts = 0.0;
  for (unsigned b = 0; b < gridDim.x; ++b) {
    td += __ldcg(partial + 2 * b);
    ts += __ldcg(partial + 2 * b + 1);
  }
  if (MODE & 4) out[0] = td;
  if (MODE & 1) out[1] = ts;
  *ticket = 0;  // ready for the next launch (stream order)
}

template <int MODE>
void launch_reduce(const double* x, double* y, uint64_t n, const double* mass_in, double* partial, unsigned* ticket,
                   double* out, cudaStream_t s) {
  const unsigned grid = (unsigned)std::min<uint64_t>(kRedBlocks, (n + kRedThreads - 1) / kRedThreads);
  iter_reduce_kernel<MODE><<<grid ? grid : 1, kRedThreads, 0, s>>>(x, y, n, mass_in, partial, ticket, out);
  note_launch();
}

}  // namespace

int iterate(const Format& f, const SpmvFn& multiply, double* x, double* work, uint32_t iters, int flags,
            double* norms, cudaStream_t s) {
  const uint64_t n = f.n;
  const bool normalize = flags & 1;
  // scratch: per-CTA partials, the ticket, and a (diff, mass) pair when the caller keeps no norms
  double* partial = nullptr;
  if (cudaMallocAsync(&partial, sizeof(double) * (2 * kRedBlocks + 2) + 64, s) != cudaSuccess) {
    cudaGetLastError();
    g_last_error = "device allocation failed (iterate scratch)";
    return kNoMemory;
  }
  double* pair = partial + 2 * kRedBlocks;
  unsigned* ticket = reinterpret_cast<unsigned*>(pair + 2);
  cudaMemsetAsync(ticket, 0, sizeof(unsigned), s);
  double* cur = x;
  double* nxt = work;
  int rc = kOk;
  for (uint32_t k = 0; k < iters && rc == kOk; ++k) {
    rc = multiply(cur, nxt, s);
    if (rc) break;
    double* out = norms ? norms + 2 * k : pair;
    if (normalize) {
      launch_reduce<1>(cur, nxt, n, nullptr, partial, ticket, out, s);     // mass of A x_k
      launch_reduce<2 | 4>(cur, nxt, n, out + 1, partial, ticket, out, s);  // rescale, then |diff|
    } else if (norms) {
      launch_reduce<1 | 4>(cur, nxt, n, nullptr, partial, ticket, out, s);
    }
    std::swap(cur, nxt);
  }
  if (rc == kOk && cur != x && n) {
    cudaMemcpyAsync(x, cur, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
  }
  cudaFreeAsync(partial, s);
  return rc ? rc : check_launch("iterate");
}

}  // namespace spmvcu
