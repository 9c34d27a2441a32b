// Device std::mt19937_64 (row A1): bit-exact with libstdc++ and therefore
// with the reference's Rng (rng.hpp:18-37).
//
// One CTA owns one engine.  The 312-word state lives in shared memory; the
// twist (libstdc++ random.tcc:399) is restated as two data-parallel phases:
//   phase A, k in [0,156):   new[k]   = old[k+156] ^ mag(old[k], old[k+1])
//   phase B, k in [156,311): new[k]   = new[k-156] ^ mag(old[k], old[k+1])
//            k = 311:        new[311] = new[155]   ^ mag(old[311], new[0])
// which is exactly the sequential in-place loop (entry k reads entry k+156
// before it is overwritten for k < 156, after it is overwritten for k >= 156).
// Tempering: random.tcc:455-470.
#pragma once

#include <stdint.h>

namespace mg {

constexpr int kMtN = 312;
constexpr int kMtM = 156;
constexpr uint64_t kMtA = 0xb5026f5aa96619e9ULL;
constexpr uint64_t kMtUpper = 0xffffffff80000000ULL;
constexpr uint64_t kMtLower = 0x000000007fffffffULL;

// splitmix64 finaliser (rng.hpp:9-14)
__host__ __device__ __forceinline__ uint64_t mg_mix64_dev(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t mt_mag(uint64_t x, uint64_t y) {
  const uint64_t z = (x & kMtUpper) | (y & kMtLower);
  return (z >> 1) ^ ((z & 1ULL) ? kMtA : 0ULL);
}

__host__ __device__ __forceinline__ uint64_t mt_temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71d67fffeda60000ULL;
  z ^= (z << 37) & 0xfff7eee000000000ULL;
  z ^= z >> 43;
  return z;
}

// rng.hpp:28: uniform in [0,1) from the top 53 bits (exact conversion).
__host__ __device__ __forceinline__ double mt_uniform(uint64_t raw) {
  return static_cast<double>(raw >> 11) * 0x1.0p-53;
}

// Seeding (libstdc++ random.tcc:328-343), sequential by definition.
__host__ __device__ inline void mt_seed(uint64_t* mt, uint64_t seed) {
  mt[0] = seed;
  for (int i = 1; i < kMtN; ++i) {
    uint64_t x = mt[i - 1];
    x ^= x >> 62;
    mt[i] = 6364136223846793005ULL * x + static_cast<uint64_t>(i);
  }
}

// Block-cooperative twist: old -> nw (distinct shared buffers).  Must be
// called by all threads of the block; blockDim.x >= 1 (any size works, 156+
// is one pass per phase).  Ends with __syncthreads().
__device__ __forceinline__ void mt_twist_block(const uint64_t* __restrict__ old,
                                               uint64_t* __restrict__ nw) {
  for (int k = threadIdx.x; k < kMtM; k += blockDim.x) nw[k] = old[k + kMtM] ^ mt_mag(old[k], old[k + 1]);
  __syncthreads();
  for (int k = kMtM + threadIdx.x; k < kMtN; k += blockDim.x) {
    if (k < kMtN - 1)
      nw[k] = nw[k - kMtM] ^ mt_mag(old[k], old[k + 1]);
    else
      nw[k] = nw[k - kMtM] ^ mt_mag(old[k], nw[0]);
  }
  __syncthreads();
}

// A block-resident engine: two shared buffers (ping-pong) + position.
struct MtBlock {
  uint64_t* buf[2];  // shared, kMtN each
  int cur;           // buffer holding the current state
  int idx;           // next output index in [0, kMtN]
};

// Loads stream state from global (row-major [kMtN]) into the block engine.
__device__ __forceinline__ void mt_block_load(MtBlock& e, const uint64_t* g_state, int g_idx) {
  for (int k = threadIdx.x; k < kMtN; k += blockDim.x) e.buf[0][k] = g_state[k];
  e.cur = 0;
  e.idx = g_idx;
  __syncthreads();
}

__device__ __forceinline__ void mt_block_store(const MtBlock& e, uint64_t* g_state, int* g_idx) {
  __syncthreads();
  for (int k = threadIdx.x; k < kMtN; k += blockDim.x) g_state[k] = e.buf[e.cur][k];
  if (threadIdx.x == 0) *g_idx = e.idx;
}

// Produces n consecutive raw outputs; calls emit(k, raw) for output k in
// [0, n) with the block's threads in parallel (k strided by blockDim).
// All threads must call.  The block's view of e stays uniform.
template <class Emit>
__device__ __forceinline__ void mt_block_generate(MtBlock& e, int64_t n, Emit emit) {
  int64_t pos = 0;
  while (pos < n) {
    if (e.idx >= kMtN) {
      mt_twist_block(e.buf[e.cur], e.buf[e.cur ^ 1]);
      e.cur ^= 1;
      e.idx = 0;
    }
    const int64_t left = n - pos;
    const int take = static_cast<int>(left < (kMtN - e.idx) ? left : (kMtN - e.idx));
    const uint64_t* st = e.buf[e.cur];
    for (int k = threadIdx.x; k < take; k += blockDim.x) emit(pos + k, mt_temper(st[e.idx + k]));
    e.idx += take;
    pos += take;
  }
  __syncthreads();
}

}  // namespace mg
