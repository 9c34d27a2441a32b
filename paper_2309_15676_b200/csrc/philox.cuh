// Philox4x32-10 counter-based generator (Salmon, Moraes, Dror, Shaw, SC'11),
// restated from the published algorithm.  Used by the scale mode of the
// samplers (mg_rng_kind MG_RNG_PHILOX): every (pixel, iteration, sample)
// gets its own counter, so any pixel's draws are computable in any thread —
// the property the sequential std::mt19937_64 stream of the reference
// (rng.hpp:36) lacks.  Statistically equivalent to the reference, not
// bit-identical; the oracle restates the same function
// (oracle/metagrad_oracle.c: mgo_philox4x32_10) for exact parity tests.
#pragma once

#include <stdint.h>

namespace mg {

struct Philox4 {
  uint32_t x[4];
};

__host__ __device__ __forceinline__ void philox_mulhilo(uint32_t a, uint32_t b, uint32_t& hi,
                                                        uint32_t& lo) {
  const uint64_t p = uint64_t(a) * uint64_t(b);
  hi = uint32_t(p >> 32);
  lo = uint32_t(p);
}

__host__ __device__ __forceinline__ Philox4 philox4x32_10(Philox4 c, uint32_t k0, uint32_t k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  constexpr uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    philox_mulhilo(M0, c.x[0], hi0, lo0);
    philox_mulhilo(M1, c.x[2], hi1, lo1);
    c = Philox4{{hi1 ^ c.x[1] ^ k0, lo1, hi0 ^ c.x[3] ^ k1, lo0}};
    k0 += W0;
    k1 += W1;
  }
  return c;
}

// Two uniform doubles in [0,1) with 53 random bits each (same conversion as
// rng.hpp:28 applied to a 53-bit integer).
__host__ __device__ __forceinline__ void philox_uniform2(Philox4 r, double& u0, double& u1) {
  const uint64_t a = (uint64_t(r.x[0]) << 21) ^ uint64_t(r.x[1] >> 11);
  const uint64_t b = (uint64_t(r.x[2]) << 21) ^ uint64_t(r.x[3] >> 11);
  u0 = double(a) * 0x1.0p-53;
  u1 = double(b) * 0x1.0p-53;
}

// Uniform s (0-based) of pixel j at iteration it, stream id st, for a
// replicate whose engine seed is key (mg_stream_seed(seed, r)).
__host__ __device__ __forceinline__ double philox_uniform_at(uint64_t key, uint32_t j, uint32_t it,
                                                             uint32_t s, uint32_t st) {
  const Philox4 r = philox4x32_10(Philox4{{j, it, s >> 1, st}}, uint32_t(key), uint32_t(key >> 32));
  double u0, u1;
  philox_uniform2(r, u0, u1);
  return (s & 1u) ? u1 : u0;
}

}  // namespace mg
