// primitives.cu -- radix sort and scan for the COO->format conversions (sm_100a).
//
// The reference sorts a permutation with a comparator (parallel_chunk_sort, inc/parallel.hpp:72-97)
// and recomputes curve ranks inside every comparison (inc/csb.hpp:77-78, inc/bcoh.hpp:240-246).
// Here every conversion first materialises one unique 64-bit key per entry and then sorts
// (key, entry index) pairs with an LSD radix sort: one "onesweep" kernel per 8-bit digit, each
// reading and writing the pairs exactly once, tile prefixes resolved by decoupled look-back.
#include <cstdio>
#include <string>

#include "common.cuh"
#include "primitives.cuh"

namespace spmvcu {

extern thread_local std::string g_last_error;

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return kCudaError;
  }
  return kOk;
}

void pool_init() {
  // Keep freed scratch in each device's default stream-ordered pool between builds instead of
  // returning it to the driver at every synchronisation (conversions allocate GBs of keys).
  once_per_device([] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t threshold = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
  });
}

void pool_trim() {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  cudaDeviceSynchronize();  // frees still in flight on other streams return to the pool first
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
}

// Stream-ordered allocation from the kept pool.  If the device is out of memory, the pool's cached
// free blocks go back to the driver (another allocator in the process -- torch's -- may need them
// as much as we do) and the allocation is retried once.
void* pool_alloc(size_t bytes, cudaStream_t s) {
  pool_init();
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, s) == cudaSuccess) return p;
  cudaGetLastError();
  pool_trim();
  if (cudaMallocAsync(&p, bytes, s) == cudaSuccess) return p;
  cudaGetLastError();
  return nullptr;
}

void* Arena::alloc(size_t bytes) {
  if (bytes == 0) bytes = 16;
  void* p = pool_alloc((bytes + 255) & ~size_t(255), s_);
  if (!p) return nullptr;
  ptrs_.push_back(p);
  return p;
}

void Arena::release() {
  for (void* p : ptrs_) cudaFreeAsync(p, s_);
  ptrs_.clear();
}

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kIpt = 16;
constexpr int kTile = kThreads * kIpt;  // 4096 pairs per tile
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPrefix = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled look-back over one 64-bit status word per (tile, lane-slot): returns the exclusive
// prefix of `count` over all earlier tiles and publishes the inclusive prefix.
__device__ __forceinline__ uint64_t lookback(uint64_t* status, uint32_t tile, uint32_t slot,
                                             uint32_t slots, uint64_t count) {
  uint64_t* mine = status + (uint64_t)tile * slots + slot;
  if (tile == 0) {
    st_relaxed(mine, kFlagPrefix | count);
    return 0;
  }
  st_relaxed(mine, kFlagAgg | count);
  uint64_t excl = 0;
  int64_t t = (int64_t)tile - 1;
  while (true) {
    const uint64_t v = ld_relaxed(status + (uint64_t)t * slots + slot);
    const uint64_t flag = v & ~kValMask;
    if (flag == 0) continue;  // predecessor not published yet
    excl += v & kValMask;
    if (flag == kFlagPrefix) break;
    --t;
  }
  st_relaxed(mine, kFlagPrefix | (excl + count));
  return excl;
}

// Warp-parallel look-back (one status word per tile; called by a whole warp): each pass inspects
// the 32 nearest unresolved predecessors at once and stops at the nearest inclusive prefix.
__device__ __forceinline__ uint64_t lookback_warp(uint64_t* status, uint32_t tile, uint64_t count,
                                                  unsigned lane) {
  uint64_t* mine = status + tile;
  if (tile == 0) {
    if (lane == 0) st_relaxed(mine, kFlagPrefix | count);
    return 0;
  }
  if (lane == 0) st_relaxed(mine, kFlagAgg | count);
  uint64_t excl = 0;
  int64_t base = (int64_t)tile - 1;
  while (true) {
    const int64_t t = base - (int64_t)lane;
    uint64_t v = t >= 0 ? ld_relaxed(status + t) : kFlagPrefix;  // before tile 0: prefix 0
    while (__any_sync(0xFFFFFFFFu, (v & ~kValMask) == 0))
      if ((v & ~kValMask) == 0) v = ld_relaxed(status + t);
    const unsigned pmask = __ballot_sync(0xFFFFFFFFu, (v & ~kValMask) == kFlagPrefix);
    const int stop = pmask ? __ffs(pmask) - 1 : 31;
    uint64_t val = (int)lane <= stop ? (v & kValMask) : 0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) val += __shfl_xor_sync(0xFFFFFFFFu, val, off);
    excl += val;
    if (pmask) break;
    base -= 32;
  }
  if (lane == 0) st_relaxed(mine, kFlagPrefix | (excl + count));
  return excl;
}

// Look-back for a tile that has ALREADY published its aggregate (flag AGG, or PREFIX for tile 0):
// walks predecessors until an inclusive prefix, then publishes its own inclusive prefix.
// Four predecessors are loaded at once (ncu: the one-at-a-time walk held 17 % of the onesweep
// kernel's stall samples on its dependent status loads).
__device__ __forceinline__ uint64_t lookback_published(uint64_t* status, uint32_t tile, uint32_t slot,
                                                       uint32_t slots, uint64_t count) {
  if (tile == 0) return 0;
  uint64_t excl = 0;
  int64_t t = (int64_t)tile - 1;
  while (true) {
    uint64_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = t - k >= 0 ? ld_relaxed(status + (uint64_t)(t - k) * slots + slot) : kFlagPrefix;
    int used = 0;
    bool done = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (done || used < k) break;
      const uint64_t flag = v[k] & ~kValMask;
      if (flag == 0) break;  // predecessor not published yet: reload from here
      excl += v[k] & kValMask;
      used = k + 1;
      done = flag == kFlagPrefix;
    }
    if (done) break;
    t -= used;
  }
  st_relaxed(status + (uint64_t)tile * slots + slot, kFlagPrefix | (excl + count));
  return excl;
}

// ------------------------------------------------------------------ radix sort

// All digit histograms in one read of the keys.  Two private copies of the [pass][digit] counts
// per CTA (warps alternate) absorb shared-atomic contention; a warp whose lanes all carry the same
// digit (the skewed high digits of power-law keys) adds 32 with one atomic.  Keys are read 4 per
// thread per step (two 128-bit loads) to keep enough bytes in flight.
constexpr int kHistCopies = 2;

__global__ void __launch_bounds__(kThreads) rs_histogram(const uint64_t* __restrict__ keys, uint64_t n,
                                                         int begin_bit, int end_bit, int npasses,
                                                         uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[kHistCopies][8 * 256];
  for (int i = threadIdx.x; i < kHistCopies * 8 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t* h = sh[warp % kHistCopies];
  auto count = [&](uint64_t key, bool valid) {
    for (int p = 0; p < npasses; ++p) {
      const int shift = begin_bit + 8 * p;
      const int bits = min(8, end_bit - shift);
      const unsigned d = (unsigned)(key >> shift) & ((1u << bits) - 1u);
      const unsigned d0 = __shfl_sync(0xFFFFFFFFu, d, 0);
      const bool same = __all_sync(0xFFFFFFFFu, valid && d == d0);
      if (same) {
        if (lane == 0) atomicAdd(&h[p * 256 + d0], 32u);
      } else if (valid) {
        atomicAdd(&h[p * 256 + d], 1u);
      }
    }
  };
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  if (reinterpret_cast<uintptr_t>(keys) & 15u) {  // unaligned caller buffer: one key per step
    for (uint64_t base = 0; base < n; base += stride) {
      const uint64_t i = base + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
      count(i < n ? keys[i] : 0, i < n);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npasses * 256; i += blockDim.x) {
      uint32_t c = 0;
      for (int k = 0; k < kHistCopies; ++k) c += sh[k][i];
      if (c) atomicAdd(&hist[i], c);
    }
    return;
  }
  const uint64_t n4 = n / 4;
  const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(keys);
  for (uint64_t base = 0; base < n4; base += stride) {  // uniform trip count across the warp
    const uint64_t i = base + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < n4;
    ulonglong2 a = make_ulonglong2(0, 0), b = make_ulonglong2(0, 0);
    if (valid) {
      a = k2[2 * i];
      b = k2[2 * i + 1];
    }
    count(a.x, valid);
    count(a.y, valid);
    count(b.x, valid);
    count(b.y, valid);
  }
  if (blockIdx.x == 0) {  // tail (n % 4 keys), warp 0
    if (warp == 0) {
      const uint64_t i = n4 * 4 + lane;
      count(i < n ? keys[i] : 0, i < n);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npasses * 256; i += blockDim.x) {
    uint32_t c = 0;
    for (int k = 0; k < kHistCopies; ++k) c += sh[k][i];
    if (c) atomicAdd(&hist[i], c);
  }
}

// hist[p][d] -> exclusive offsets over d, in place.  One block per pass.
__global__ void rs_hist_scan(uint32_t* hist) {
  __shared__ uint32_t s[256];
  uint32_t* h = hist + blockIdx.x * 256;
  s[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int d = 0; d < 256; ++d) {
      const uint32_t c = s[d];
      s[d] = run;
      run += c;
    }
  }
  __syncthreads();
  h[threadIdx.x] = s[threadIdx.x];
}

// Pairs per thread (IPT): only the keys are live in registers while ranking, which keeps the
// kernel small enough for 3 CTAs per SM.  The tile's values never pass through registers before
// the write-out: one thread starts a bulk async copy (cp.async.bulk + mbarrier) of the tile's
// value range into shared memory as soon as the tile index is known, overlapping the key loads
// and the ranking; the keys are staged in digit order as 32-bit halves with their 16-bit
// position in the tile, which the write-out uses to fetch the value.
template <typename V>
struct OneSweep {
  static constexpr int IPT = 12;
  static constexpr int TILE = kThreads * IPT;
  static constexpr size_t SMEM = sizeof(V) * TILE + sizeof(uint32_t) * TILE * 2 + sizeof(uint16_t) * TILE +
                                 sizeof(uint32_t) * kWarps * 256 + sizeof(uint32_t) * 256 + sizeof(int64_t) * 256;
};

template <typename V>
__global__ void __launch_bounds__(kThreads, 3) rs_onesweep(
    const uint64_t* __restrict__ kin, const V* __restrict__ vin, uint64_t* __restrict__ kout,
    V* __restrict__ vout, uint64_t n, int shift, uint32_t dmask,
    const uint32_t* __restrict__ pass_offset, uint64_t* status, uint32_t* tile_counter) {
  constexpr int kIpt = OneSweep<V>::IPT;
  constexpr int kTile = OneSweep<V>::TILE;
  extern __shared__ __align__(128) uint8_t smem[];
  V* s_vorig = reinterpret_cast<V*>(smem);                      // values in input order (bulk copy)
  uint32_t* s_klo = reinterpret_cast<uint32_t*>(s_vorig + kTile);
  uint32_t* s_khi = s_klo + kTile;
  uint16_t* s_pos = reinterpret_cast<uint16_t*>(s_khi + kTile);  // input position of each staged key
  uint32_t* s_whist = reinterpret_cast<uint32_t*>(s_pos + kTile);  // [warp][digit]
  uint32_t* s_local = s_whist + kWarps * 256;       // tile-local exclusive digit offsets
  int64_t* s_gbase = reinterpret_cast<int64_t*>(s_local + 256);
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_wsum[kWarps];
  __shared__ __align__(8) uint64_t s_bar;

  const unsigned tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
  if (tid == 0) {
    const uint32_t t = atomicAdd(tile_counter, 1u);
    s_tile = t;
    mbar_init(&s_bar, 1);
    fence_mbar_init();
    const uint64_t b0 = (uint64_t)t * kTile;
    const uint32_t cnt0 = (n - b0) < (uint64_t)kTile ? (uint32_t)(n - b0) : (uint32_t)kTile;
    const bool aligned = (reinterpret_cast<uintptr_t>(vin) & 15u) == 0;
    const uint32_t bytes = aligned ? (cnt0 * (uint32_t)sizeof(V)) & ~15u : 0u;  // 16-B multiple; rest below
    mbar_arrive_expect_tx(&s_bar, bytes);
    if (bytes) bulk_g2s(s_vorig, vin + b0, bytes, &s_bar, policy_evict_first());
  }
  for (int i = tid; i < kWarps * 256; i += kThreads) s_whist[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = (uint64_t)tile * kTile;
  const uint64_t wbase = base + (uint64_t)warp * (kIpt * 32);
  const uint32_t valid_n = (n - base) < (uint64_t)kTile ? (uint32_t)(n - base) : (uint32_t)kTile;
  {  // the values the 16-byte bulk copy leaves out (a few trailing ones; all if vin is unaligned)
    const bool aligned = (reinterpret_cast<uintptr_t>(vin) & 15u) == 0;
    const uint32_t done = aligned ? (valid_n * (uint32_t)sizeof(V) & ~15u) / (uint32_t)sizeof(V) : 0u;
    for (uint32_t q = done + tid; q < valid_n; q += kThreads) s_vorig[q] = vin[base + q];
  }

  uint64_t key[kIpt];
  uint32_t rank[kIpt];
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const uint64_t idx = wbase + i * 32 + lane;
    key[i] = idx < n ? kin[idx] : 0;
  }
  const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const uint64_t idx = wbase + i * 32 + lane;
    const bool valid = idx < n;
    const unsigned d = valid ? ((unsigned)(key[i] >> shift) & dmask) : (0x100u + lane);
    // (8 per-bit ballots instead of match.any measured no faster on sm_100: 797 vs 793 us/pass)
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
    uint32_t prior = 0;
    if (valid) {
      prior = s_whist[warp * 256 + d];
      rank[i] = prior + __popc(peers & lt_mask);
    }
    __syncwarp();
    if (valid && lane == (unsigned)(__ffs(peers) - 1)) s_whist[warp * 256 + d] = prior + __popc(peers);
    __syncwarp();
  }
  __syncthreads();

  // per digit (one thread each): warp prefix, tile count, tile-local offset, global base
  const unsigned d = tid;
  uint32_t cnt = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const uint32_t c = s_whist[w * 256 + d];
    s_whist[w * 256 + d] = cnt;
    cnt += c;
  }
  // block-exclusive scan of cnt over digits
  uint32_t incl = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
    if (lane >= (unsigned)off) incl += t;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  uint32_t wpre = 0;
  for (unsigned w = 0; w < warp; ++w) wpre += s_wsum[w];
  const uint32_t local_excl = wpre + incl - cnt;
  // fold the tile-local digit offset into every warp's prefix: pos = s_whist[warp][d] + rank
#pragma unroll
  for (int w = 0; w < kWarps; ++w) s_whist[w * 256 + d] += local_excl;
  // publish this tile's counts before doing local work so successors can proceed
  uint64_t* mine = status + (uint64_t)tile * 256 + d;
  st_relaxed(mine, (tile == 0 ? kFlagPrefix : kFlagAgg) | cnt);
  __syncthreads();

  // stage the keys in digit order in shared memory (needs only tile-local offsets)
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const uint32_t li = warp * (kIpt * 32) + i * 32 + lane;
    if (base + li < n) {
      const unsigned dd = (unsigned)(key[i] >> shift) & dmask;
      const uint32_t pos = s_whist[warp * 256 + dd] + rank[i];
      s_klo[pos] = (uint32_t)key[i];
      s_khi[pos] = (uint32_t)(key[i] >> 32);
      s_pos[pos] = (uint16_t)li;
    }
  }
  // ... then resolve the global offsets by look-back (overlapping predecessors' progress)
  const uint64_t excl = lookback_published(status, tile, d, 256, cnt);
  s_gbase[d] = (int64_t)pass_offset[d] + (int64_t)excl - (int64_t)local_excl;
  __syncthreads();
  mbar_wait(&s_bar, 0);  // the tile's values have landed
  for (uint32_t j = tid; j < valid_n; j += kThreads) {
    const uint64_t k = ((uint64_t)s_khi[j] << 32) | s_klo[j];
    const unsigned dd = (unsigned)(k >> shift) & dmask;
    const uint64_t o = (uint64_t)(s_gbase[dd] + (int64_t)j);
    kout[o] = k;
    vout[o] = s_vorig[s_pos[j]];
  }
}

// ------------------------------------------------------------------ exclusive scan

__device__ __forceinline__ unsigned pad_idx(unsigned i) { return i + (i >> 5); }

__global__ void __launch_bounds__(kThreads) scan_u32(const uint32_t* in, uint32_t* out, uint64_t n,
                                                     uint64_t* status, uint32_t* tile_counter) {
  __shared__ uint32_t s[kTile + kTile / 32];
  __shared__ uint32_t s_wsum[kWarps];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_excl;
  const unsigned tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = (uint64_t)tile * kTile;
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const unsigned li = i * kThreads + tid;
    const uint64_t idx = base + li;
    s[pad_idx(li)] = idx < n ? in[idx] : 0u;
  }
  __syncthreads();
  uint32_t v[kIpt];
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < kIpt; ++k) {
    v[k] = s[pad_idx(tid * kIpt + k)];
    sum += v[k];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, off);
    if (lane >= (unsigned)off) incl += t;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  uint32_t wpre = 0, total = 0;
  for (int w = 0; w < kWarps; ++w) {
    if ((unsigned)w < warp) wpre += s_wsum[w];
    total += s_wsum[w];
  }
  if (warp == 0) {
    const uint64_t ex = lookback_warp(status, tile, total, lane);
    if (lane == 0) s_excl = ex;
  }
  __syncthreads();
  uint32_t run = (uint32_t)s_excl + wpre + incl - sum;
#pragma unroll
  for (int k = 0; k < kIpt; ++k) {
    s[pad_idx(tid * kIpt + k)] = run;
    run += v[k];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const unsigned li = i * kThreads + tid;
    const uint64_t idx = base + li;
    if (idx < n) out[idx] = s[pad_idx(li)];
  }
  if (base + kTile >= n && tid == 0) out[n] = (uint32_t)(s_excl + total);
}

}  // namespace

template <typename V>
bool radix_sort_pairs(uint64_t* keys, uint64_t* keys_alt, V* vals, V* vals_alt,
                      uint64_t n, int begin_bit, int end_bit, Arena& arena) {
  if (n <= 1 || end_bit <= begin_bit) return false;
  cudaStream_t s = arena.stream();
  const int npasses = (end_bit - begin_bit + 7) / 8;
  uint32_t* hist = arena.alloc_n<uint32_t>(npasses * 256);
  cudaMemsetAsync(hist, 0, sizeof(uint32_t) * npasses * 256, s);
  const int hblocks = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)kNumSMs * 8);
  rs_histogram<<<hblocks, 256, 0, s>>>(keys, n, begin_bit, end_bit, npasses, hist);
  rs_hist_scan<<<npasses, 256, 0, s>>>(hist);

  const uint64_t tiles = (n + OneSweep<V>::TILE - 1) / OneSweep<V>::TILE;
  uint64_t* status = arena.alloc_n<uint64_t>(tiles * 256 + 8);
  uint32_t* counter = reinterpret_cast<uint32_t*>(status + tiles * 256);
  constexpr size_t smem = OneSweep<V>::SMEM;
  once_per_device(
      [] { cudaFuncSetAttribute(rs_onesweep<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
  bool in_alt = false;
  for (int p = 0; p < npasses; ++p) {
    const int shift = begin_bit + 8 * p;
    const int bits = std::min(8, end_bit - shift);
    cudaMemsetAsync(status, 0, sizeof(uint64_t) * (tiles * 256 + 8), s);
    const uint64_t* ki = in_alt ? keys_alt : keys;
    const V* vi = in_alt ? vals_alt : vals;
    uint64_t* ko = in_alt ? keys : keys_alt;
    V* vo = in_alt ? vals : vals_alt;
    rs_onesweep<V><<<(unsigned)tiles, kThreads, smem, s>>>(ki, vi, ko, vo, n, shift, (1u << bits) - 1u,
                                                           hist + p * 256, status, counter);
    in_alt = !in_alt;
  }
  return in_alt;
}

template bool radix_sort_pairs<uint32_t>(uint64_t*, uint64_t*, uint32_t*, uint32_t*, uint64_t, int, int, Arena&);
template bool radix_sort_pairs<uint64_t>(uint64_t*, uint64_t*, uint64_t*, uint64_t*, uint64_t, int, int, Arena&);

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, Arena& arena) {
  cudaStream_t s = arena.stream();
  if (n == 0) {
    cudaMemsetAsync(out, 0, sizeof(uint32_t), s);
    return;
  }
  const uint64_t tiles = (n + kTile - 1) / kTile;
  uint64_t* status = arena.alloc_n<uint64_t>(tiles + 8);
  cudaMemsetAsync(status, 0, sizeof(uint64_t) * (tiles + 8), s);
  scan_u32<<<(unsigned)tiles, kThreads, 0, s>>>(in, out, n, status,
                                                reinterpret_cast<uint32_t*>(status + tiles));
}

}  // namespace spmvcu
