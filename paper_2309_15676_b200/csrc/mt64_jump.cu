// Jump-ahead for std::mt19937_64 (row A1 at scale).
//
// The reference's stream (rng.hpp:36) is sequential: output t needs t
// twists.  To let many CTAs produce disjoint segments of ONE replicate's
// stream bit-exactly (a single large mini-render replicate draws P*spp
// uniforms per iteration, problems.cpp:201-202), each engine is advanced by
// a fixed distance J with the GF(2) jump-ahead method (Haramoto, Matsumoto,
// Nishimura, Panneton, L'Ecuyer, "Efficient jump ahead for F2-linear random
// number generators", 2008), restated here:
//
//   * the per-output state transition A of the 19937-dimensional generator
//     has characteristic polynomial phi(x) (degree 19937); it is recovered
//     once from 2*19937 output bits with Berlekamp-Massey;
//   * g(x) = x^J mod phi(x) by square-and-multiply;
//   * the jumped state is g(A) s, evaluated by Horner's rule on the state
//     "window" (x_t .. x_{t+311}) with 4-bit digits on the device
//     (mt64.cu: mt_jump_kernel).
//
// All host code; polynomials are little-endian bit arrays in uint64 words.
#include <stdint.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "mg_common.cuh"
#include "mt64.cuh"
#include "mt64_jump.h"

namespace mg {
namespace {

using Poly = std::vector<uint64_t>;
constexpr int kDeg = 19937;              // degree of phi
constexpr int kWords = (kDeg + 63) / 64;  // residues mod phi: 312 words

inline int getbit(const Poly& p, int i) { return int((p[size_t(i) >> 6] >> (i & 63)) & 1u); }
inline void flipbit(Poly& p, int i) { p[size_t(i) >> 6] ^= 1ULL << (i & 63); }

// p ^= q << shift   (q has qbits significant bits)
void xor_shifted(Poly& p, const Poly& q, int qwords, int shift) {
  const int ws = shift >> 6, bs = shift & 63;
  for (int i = 0; i < qwords; ++i) {
    const uint64_t w = q[size_t(i)];
    if (!w) continue;
    p[size_t(i + ws)] ^= w << bs;
    if (bs && size_t(i + ws + 1) < p.size()) p[size_t(i + ws + 1)] ^= w >> (64 - bs);
  }
}

// Output bits of the generator, one per output (bit 0 of each raw output):
// a linear functional of the state, so its minimal polynomial is phi.
std::vector<uint8_t> output_bits(int n) {
  std::vector<uint64_t> mt(kMtN);
  mt_seed(mt.data(), 5489ULL);
  std::vector<uint8_t> bits(static_cast<size_t>(n));
  int idx = kMtN;
  for (int t = 0; t < n; ++t) {
    if (idx >= kMtN) {
      for (int k = 0; k < kMtN; ++k)
        mt[size_t(k)] = mt[size_t((k + kMtM) % kMtN)] ^ mt_mag(mt[size_t(k)], mt[size_t((k + 1) % kMtN)]);
      idx = 0;
    }
    bits[size_t(t)] = uint8_t(mt_temper(mt[size_t(idx++)]) & 1u);
  }
  return bits;
}

// Berlekamp-Massey over GF(2): connection polynomial C (c_0 = 1) of the
// shortest LFSR generating s; returns phi(x) = x^L C(1/x).
Poly characteristic_polynomial() {
  const int N = 2 * kDeg + 64;
  const std::vector<uint8_t> s = output_bits(N);
  const int W = (N + 63) / 64 + 2;
  Poly C(size_t(W), 0), B(size_t(W), 0), T;
  C[0] = B[0] = 1;
  int L = 0, m = 1;
  // reversed sequence bits for fast discrepancy: rev bit k = s[N-1-k]
  Poly rev(size_t(W), 0);
  for (int k = 0; k < N; ++k)
    if (s[size_t(N - 1 - k)]) rev[size_t(k) >> 6] |= 1ULL << (k & 63);
  for (int n = 0; n < N; ++n) {
    // d = sum_{i=0..L} c_i s_{n-i} = parity(C & (rev >> (N-1-n)))
    const int off = N - 1 - n;
    uint64_t acc = 0;
    const int cw = L / 64 + 1;
    const int ow = off >> 6, ob = off & 63;
    for (int i = 0; i < cw; ++i) {
      uint64_t r = rev[size_t(ow + i)] >> ob;
      if (ob && size_t(ow + i + 1) < rev.size()) r |= rev[size_t(ow + i + 1)] << (64 - ob);
      acc ^= C[size_t(i)] & r;
    }
    const int d = __builtin_parityll(acc);
    if (!d) {
      ++m;
    } else if (2 * L <= n) {
      T = C;
      xor_shifted(C, B, W - (m >> 6) - 1, m);
      L = n + 1 - L;
      B = T;
      m = 1;
    } else {
      xor_shifted(C, B, W - (m >> 6) - 1, m);
      ++m;
    }
  }
  Poly phi(size_t(kWords + 1), 0);  // degree L needs L+1 bits
  for (int i = 0; i <= L; ++i)
    if (getbit(C, i)) flipbit(phi, L - i);
  if (L != kDeg) phi.clear();  // not the expected generator
  return phi;
}

std::once_flag g_phi_once;
Poly g_phi;

const Poly& phi() {
  std::call_once(g_phi_once, [] { g_phi = characteristic_polynomial(); });
  return g_phi;
}

// r = r mod phi, r holding up to 2*kDeg bits
void reduce(Poly& r, const Poly& f) {
  for (int k = 2 * kDeg; k >= kDeg; --k)
    if (getbit(r, k)) xor_shifted(r, f, kWords + 1, k - kDeg);
}

Poly square_mod(const Poly& a, const Poly& f) {
  Poly r(size_t(2 * kWords + 2), 0);
  for (int i = 0; i < kDeg; ++i)
    if (getbit(a, i)) flipbit(r, 2 * i);
  reduce(r, f);
  r.resize(size_t(kWords));
  return r;
}

Poly times_x_mod(const Poly& a, const Poly& f) {
  Poly r(size_t(kWords + 1), 0);
  for (int i = 0; i < kWords; ++i) {
    r[size_t(i)] |= a[size_t(i)] << 1;
    r[size_t(i + 1)] |= a[size_t(i)] >> 63;
  }
  if (getbit(r, kDeg)) xor_shifted(r, f, kWords + 1, 0);
  r.resize(size_t(kWords));
  return r;
}

}  // namespace

bool mt64_jump_polynomial(uint64_t distance, uint64_t* out_words, int* out_deg) {
  const Poly& f = phi();
  if (f.empty()) return false;
  Poly r(size_t(kWords), 0);
  r[0] = 1;  // x^0
  int top = 63;
  while (top >= 0 && !((distance >> top) & 1u)) --top;
  for (int b = top; b >= 0; --b) {
    r = square_mod(r, f);
    if ((distance >> b) & 1u) r = times_x_mod(r, f);
  }
  int deg = -1;
  for (int i = kDeg - 1; i >= 0; --i)
    if (getbit(r, i)) {
      deg = i;
      break;
    }
  memcpy(out_words, r.data(), sizeof(uint64_t) * kWords);
  *out_deg = deg;
  return true;
}

int mt64_char_poly(uint64_t* out_words /* kWords+1 */) {
  const Poly& f = phi();
  if (f.empty()) return MG_ECUDA;
  memcpy(out_words, f.data(), sizeof(uint64_t) * (kWords + 1));
  return MG_OK;
}

}  // namespace mg

extern "C" int mg_mt64_jump_polynomial(uint64_t distance, uint64_t* out_words, int32_t* out_deg) {
  if (!out_words || !out_deg) return mg::fail(MG_EINVAL, "mg_mt64_jump_polynomial: null argument");
  int deg = 0;
  if (!mg::mt64_jump_polynomial(distance, out_words, &deg))
    return mg::fail(MG_ELOGIC, "mt19937_64 characteristic polynomial: unexpected degree");
  *out_deg = deg;
  return MG_OK;
}
