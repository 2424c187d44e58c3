// primitives.cuh -- device-wide building blocks for the conversions (hand-written, sm_100a):
//   * LSD radix sort of (u64 key, u32 value) pairs, one "onesweep" pass per 8-bit digit with
//     decoupled look-back (one read + one write of the pairs per digit);
//   * exclusive scan of u32 counts with decoupled look-back (row_ptr / blk_ptr construction);
//   * a stream-ordered scratch arena.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <mutex>
#include <vector>

namespace spmvcu {

// Stream-ordered scratch allocations released when the arena dies.
// Keeps freed device memory in the default stream-ordered pool (release threshold = max).
void pool_init();
void pool_trim();                             // return the pool's cached free blocks to the driver
void* pool_alloc(size_t bytes, cudaStream_t s);  // cudaMallocAsync, trim + retry once when out of memory

class Arena {
 public:
  explicit Arena(cudaStream_t s) : s_(s) {}
  ~Arena() { release(); }
  void* alloc(size_t bytes);
  template <typename T>
  T* alloc_n(size_t n) { return static_cast<T*>(alloc(n * sizeof(T))); }
  void release();
  cudaStream_t stream() const { return s_; }

 private:
  cudaStream_t s_;
  std::vector<void*> ptrs_;
};

// Sorts n pairs by key bits [begin_bit, end_bit).  Stable.  Uses keys_alt/vals_alt as ping-pong
// buffers; returns true if the result ended in the *_alt buffers.
// V = uint32_t (an index payload) or uint64_t (a value's bit pattern carried through the sort).
template <typename V>
bool radix_sort_pairs(uint64_t* keys, uint64_t* keys_alt, V* vals, V* vals_alt,
                      uint64_t n, int begin_bit, int end_bit, Arena& arena);

// out[0..n] = exclusive prefix sums of in[0..n); out[n] = total.  in and out may alias.
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, Arena& arena);

// Launch-error check helper: returns 0 or kCudaError and records the message.
int check_launch(const char* what);

// Runs `setup` once per (call site, current device), thread-safe: kernel attributes such as the
// dynamic shared-memory limit are per device, and a concurrent first launch must not race ahead
// of them.
template <typename F>
inline void once_per_device(F&& setup) {
  static std::mutex mu;
  static uint64_t done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  std::lock_guard<std::mutex> lk(mu);
  if (!(done & bit)) {
    setup();
    done |= bit;
  }
}

}  // namespace spmvcu
