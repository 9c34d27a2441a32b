// Host-side jump polynomials for std::mt19937_64 (mt64_jump.cu).
#pragma once
#include <stdint.h>

namespace mg {
constexpr int kMtJumpWords = 312;  // residues mod phi (degree 19937)
// g(x) = x^distance mod phi(x); out_words[kMtJumpWords]; deg of g (-1: g = 0)
bool mt64_jump_polynomial(uint64_t distance, uint64_t* out_words, int* out_deg);
int mt64_char_poly(uint64_t* out_words /* kMtJumpWords + 1 */);
}  // namespace mg
