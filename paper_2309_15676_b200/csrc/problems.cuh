// Per-sample device math of the reference problems (rows A3, A6, A7),
// shared by the standalone sample_pair kernels and the fused runner.
#pragma once

#include <math.h>

namespace mg {

// Vectors up to this size are reduced sequentially by one thread, which is
// bit-identical to the reference's squaredNorm()/sum() (sequential under the
// shim); larger ones use a fixed-order tree (deterministic, tolerance-equal).
constexpr int kSeqReduceMax = 4096;

// MiniRenderProblem::kernel_terms for one pixel (problems.cpp:177-195).
// fp64: the reference's expression order exactly.
// fp32: the algebraically identical pairwise form
//   cross = 2 * sum_{s<t} basis_s basis_t / (n (n-1))
// which has no cancellation (all terms >= 0); the reference's
// (sum^2 - sum_sq) loses up to 1e-3 relative in fp32 when one sample
// dominates.  See DESIGN.md "fp32 sampling".
template <class T>
__device__ __forceinline__ void minirender_terms(double b, const double* __restrict__ u, int spp,
                                                 T& cross, T& mean_basis);

template <>
__device__ __forceinline__ void minirender_terms<double>(double b, const double* __restrict__ u,
                                                         int spp, double& cross,
                                                         double& mean_basis) {
  const double n = double(spp);
  double sum = 0.0, sum_sq = 0.0;
  for (int s = 0; s < spp; ++s) {
    const double basis = (b + 1.0) * pow(u[s], b);
    sum += basis;
    sum_sq += basis * basis;
  }
  cross = (sum * sum - sum_sq) / (n * (n - 1.0));
  mean_basis = sum / n;
}

template <>
__device__ __forceinline__ void minirender_terms<float>(double b, const double* __restrict__ u,
                                                        int spp, float& cross, float& mean_basis) {
  const float n = float(spp);
  const float bf = float(b);
  float sum = 0.f, pairs = 0.f;
  for (int s = 0; s < spp; ++s) {
    const float basis = (bf + 1.f) * powf(float(u[s]), bf);
    pairs += basis * sum;
    sum += basis;
  }
  cross = (2.f * pairs) / (n * (n - 1.f));
  mean_basis = sum / n;
}

// Same terms with the uniforms supplied by a functor u(s) (fused kernels).
template <class T, class U>
__device__ __forceinline__ void minirender_terms_fn(double b, int spp, U u, T& cross,
                                                    T& mean_basis) {
  if constexpr (sizeof(T) == 8) {
    const double n = double(spp);
    double sum = 0.0, sum_sq = 0.0;
    for (int s = 0; s < spp; ++s) {
      const double basis = (b + 1.0) * pow(u(s), b);
      sum += basis;
      sum_sq += basis * basis;
    }
    cross = (sum * sum - sum_sq) / (n * (n - 1.0));
    mean_basis = sum / n;
  } else {
    const float n = float(spp);
    const float bf = float(b);
    float sum = 0.f, pairs = 0.f;
    for (int s = 0; s < spp; ++s) {
      const float basis = (bf + 1.f) * powf(float(u(s)), bf);
      pairs += basis * sum;
      sum += basis;
    }
    cross = (2.f * pairs) / (n * (n - 1.f));
    mean_basis = sum / n;
  }
}

// fp32 fast-mode u^b for u in [0,1), b >= 0: exp2(b * log2(u)) on the SFU
// (MUFU.LG2 / MUFU.EX2).  |log2 u| <= 53 and b <= exponent_max keep the
// relative error ~1e-6 (tolerance 1e-4); pow(u, 0) = 1 and
// pow(0, b>0) = 0 as in libm.
__device__ __forceinline__ float fast_powf01(float u, float b) {
  if (b == 0.f) return 1.f;
  if (u == 0.f) return 0.f;
  return exp2f(b * __log2f(u));
}

// Same terms from a register array of up to MAXS uniforms (spp <= MAXS),
// fully unrolled so the array stays in registers.
template <class T, int MAXS>
__device__ __forceinline__ void minirender_terms_arr(double b, int spp, const double (&u)[MAXS],
                                                     T& cross, T& mean_basis) {
  if constexpr (sizeof(T) == 8) {
    const double n = double(spp);
    double sum = 0.0, sum_sq = 0.0;
#pragma unroll
    for (int s = 0; s < MAXS; ++s) {
      if (s < spp) {
        const double basis = (b + 1.0) * pow(u[s], b);
        sum += basis;
        sum_sq += basis * basis;
      }
    }
    cross = (sum * sum - sum_sq) / (n * (n - 1.0));
    mean_basis = sum / n;
  } else {
    const float n = float(spp);
    const float bf = float(b);
    float sum = 0.f, pairs = 0.f;
#pragma unroll
    for (int s = 0; s < MAXS; ++s) {
      if (s < spp) {
        const float basis = (bf + 1.f) * fast_powf01(float(u[s]), bf);
        pairs += basis * sum;
        sum += basis;
      }
    }
    cross = (2.f * pairs) / (n * (n - 1.f));
    mean_basis = sum / n;
  }
}

// ExpRateProblem draws (problems.cpp:58-63); u are uniform_pos() values.
__device__ __forceinline__ void exprate_sums(const double* __restrict__ u, int n, double& sum_c,
                                             double& sum_c_sq) {
  for (int k = 0; k < n; ++k) {
    const double c = -log(u[k]);
    sum_c += c;
    sum_c_sq += c * c;
  }
}

// ExpRateProblem::gradient_from_batch (problems.cpp:44-52)
__device__ __forceinline__ double exprate_gradient(double target_mean, int samples, double rate,
                                                   double sum_c, double sum_c_sq) {
  const double n = double(samples);
  const double rate_sq = rate * rate;
  return ((-2.0) * (sum_c * sum_c - sum_c_sq)) / (((n * (n - 1.0)) * rate_sq) * rate) +
         ((2.0 * target_mean) * sum_c) / (n * rate_sq);
}

// MultNoiseQuadratic::noise_factors_from_draws for coordinate j
// (problems.cpp:110-119): sample-major uniforms u[s*d + j].
__device__ __forceinline__ double multnoise_factor(const double* __restrict__ u, int d, int n,
                                                   int j, double sigma) {
  double f = 0.0;
  for (int s = 0; s < n; ++s) f += 1.0 + sigma * (2.0 * u[size_t(s) * d + j] - 1.0);
  return f / double(n);
}

}  // namespace mg
