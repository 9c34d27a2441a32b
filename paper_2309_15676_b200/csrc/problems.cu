// Gradient-sample sources (rows A2-A7): the reference's three synthetic
// problems, batched over replicates.  Each replicate r consumes its own
// std::mt19937_64 stream exactly as the reference's sample_pair does
// (problems.cpp:201-202, :58-63, :125-126), so in fp64 mode the draws are
// bit-identical and every output is the reference's expression evaluated in
// the same operation order (transcendentals: CUDA pow/log).
#include <math.h>

#include "mg_common.cuh"
#include "mt64.cuh"
#include "mt64_state.h"
#include "problems.cuh"

namespace mg {
namespace {

constexpr int kThreads = 256;

// problems.cpp:168-172: b_j = exponent_max * u_j (first P draws), then
// T_j = 0.2 + 0.8 * u_{P+j}.  In place over the two uniform blocks.
__global__ void minirender_gen_kernel(int P, double exponent_max, double* __restrict__ b,
                                      double* __restrict__ T) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P; j += gridDim.x * blockDim.x) {
    b[j] = exponent_max * b[j];
    T[j] = 0.2 + 0.8 * T[j];
  }
}

// Per replicate: ssn = sum (now - prev)^2 and changed = #(now != prev).
// Small vectors are summed sequentially (bit-identical to the reference's
// squaredNorm under the shim); larger ones with a fixed tree.
template <class T>
__global__ void pair_norm_kernel(int R, int P, const T* __restrict__ now,
                                 const T* __restrict__ prev, double* __restrict__ ssn,
                                 int* __restrict__ changed) {
  __shared__ double sw[kThreads / 32];
  const int r = blockIdx.x;
  const T* a = now + size_t(r) * P;
  const T* b = prev + size_t(r) * P;
  if (P <= kSeqReduceMax) {
    if (threadIdx.x == 0) {
      double s = 0.0;
      int c = 0;
      for (int j = 0; j < P; ++j) {
        const double d = double(a[j] - b[j]);
        s += d * d;
        c += (a[j] != b[j]);
      }
      ssn[r] = s;
      changed[r] = c;
    }
    return;
  }
  double s = 0.0, c = 0.0;
  for (int j = threadIdx.x; j < P; j += kThreads) {
    const double d = double(a[j] - b[j]);
    s += d * d;
    c += (a[j] != b[j]) ? 1.0 : 0.0;
  }
  s = block_sum<kThreads>(s, sw);
  c = block_sum<kThreads>(c, sw);
  if (threadIdx.x == 0) {
    ssn[r] = s;
    changed[r] = int(c);
  }
}

// problems.cpp:197-217 per pixel, grid (pixel blocks, R).
template <class T>
__global__ void minirender_pair_kernel(int R, int P, int spp, const double* __restrict__ b,
                                       const double* __restrict__ tgt,
                                       const double* __restrict__ u, const T* __restrict__ now,
                                       const T* __restrict__ prev, T* __restrict__ prop,
                                       T* __restrict__ diff, double* __restrict__ ssn,
                                       const int* __restrict__ changed) {
  for (int r = blockIdx.y; r < R; r += gridDim.y) {
  const bool same = changed[r] == 0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P; j += gridDim.x * blockDim.x) {
    const size_t at = size_t(r) * P + j;
    T cross, mb;
    minirender_terms<T>(b[j], u + size_t(r) * P * spp + size_t(j) * spp, spp, cross, mb);
    const T a = now[at];
    prop[at] = (T(2) * a) * cross - (T(2) * T(tgt[j])) * mb;  // :205
    diff[at] = same ? T(0) : (T(2) * (a - prev[at])) * cross;  // :206-213
  }
  if (same && blockIdx.x == 0 && threadIdx.x == 0) ssn[r] = 0.0;  // :208
  }
}

// problems.cpp:54-76 (dim 1): one thread per replicate, sequential sums.
__global__ void exprate_pair_kernel(int R, int n, double target_mean, const double* __restrict__ u,
                                    const double* __restrict__ now,
                                    const double* __restrict__ prev, double* __restrict__ prop,
                                    double* __restrict__ diff, double* __restrict__ ssn) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  double sum_c = 0.0, sum_c_sq = 0.0;
  exprate_sums(u + size_t(r) * n, n, sum_c, sum_c_sq);
  const double rn = now[r], rp = prev[r];
  const double g = exprate_gradient(target_mean, n, rn, sum_c, sum_c_sq);
  prop[r] = g;
  if (rn == rp) {
    diff[r] = 0.0;
    ssn[r] = 0.0;
  } else {
    diff[r] = g - exprate_gradient(target_mean, n, rp, sum_c, sum_c_sq);
    ssn[r] = (rn - rp) * (rn - rp);
  }
}

// problems.cpp:110-139, one thread per replicate (dims are tiny).
__global__ void multnoise_pair_kernel(int R, int d, int n, double sigma,
                                      const double* __restrict__ target,
                                      const double* __restrict__ u,
                                      const double* __restrict__ now,
                                      const double* __restrict__ prev, double* __restrict__ prop,
                                      double* __restrict__ diff, double* __restrict__ ssn) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const double* ur = u + size_t(r) * d * n;
  const double* a = now + size_t(r) * d;
  const double* p = prev + size_t(r) * d;
  bool same = true;
  for (int j = 0; j < d; ++j) same &= (a[j] == p[j]);
  double s = 0.0;
  for (int j = 0; j < d; ++j) {
    const double f = multnoise_factor(ur, d, n, j, sigma);
    prop[size_t(r) * d + j] = (a[j] - target[j]) * f;
    if (same) {
      diff[size_t(r) * d + j] = 0.0;
    } else {
      const double dj = a[j] - p[j];
      diff[size_t(r) * d + j] = dj * f;
      s += dj * dj;
    }
  }
  ssn[r] = same ? 0.0 : s;
}

__global__ void domain_check_kernel(int R, const double* __restrict__ a,
                                    const double* __restrict__ b, int* flag) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R && (!(a[r] > 0.0) || !(b[r] > 0.0))) *flag = 1;  // problems.cpp:93
}

}  // namespace
}  // namespace mg

using namespace mg;

extern "C" {

int mg_minirender_generate(mg_ctx* ctx, int32_t pixel_count, uint64_t gen_seed, double exponent_max,
                           double* exponents, double* target) {
  if (!ctx || !exponents || !target) return fail(MG_EINVAL, "mg_minirender_generate: null argument");
  if (pixel_count < 1) return fail(MG_EINVAL, "mini-render: pixel_count must be >= 1");
  if (!(exponent_max >= 0.0)) return fail(MG_EINVAL, "mini-render: exponent_max must be >= 0");
  const uint64_t seed = mg_mix64(gen_seed);  // Rng gen(mix64(gen_seed)), problems.cpp:168
  mg_mt64* g = nullptr;
  int st = mt64_create(ctx, 1, &seed, &g);
  if (st) return st;
  st = mt64_draw(ctx, g, pixel_count, 1, exponents);
  if (!st) st = mt64_draw(ctx, g, pixel_count, 1, target);
  if (!st) {
    minirender_gen_kernel<<<grid_for(ctx, pixel_count, 256, 4), 256, 0, ctx->stream>>>(
        pixel_count, exponent_max, exponents, target);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) st = cuda_fail(e, "minirender_gen_kernel");
  }
  cudaStreamSynchronize(ctx->stream);
  mt64_destroy(g);
  return st;
}

int mg_minirender_sample_pair(mg_ctx* ctx, int32_t dtype, int32_t R, int32_t P, int32_t spp,
                              const double* exponents, const double* target, mg_mt64* g,
                              const void* now, const void* prev, void* prop, void* diff,
                              double* ssn_out) {
  if (!ctx || !g || !exponents || !target || !now || !prev || !prop || !diff || !ssn_out)
    return fail(MG_EINVAL, "mg_minirender_sample_pair: null argument");
  if (spp < 2) return fail(MG_EINVAL, "mini-render: spp must be at least 2");
  if (P < 1 || R < 1 || R > g->streams) return fail(MG_EINVAL, "mg_minirender_sample_pair: bad sizes");
  double* u = nullptr;
  int* changed = nullptr;
  MG_CUDA_TRY(cudaMallocAsync(&u, sizeof(double) * size_t(R) * P * spp, ctx->stream));
  MG_CUDA_TRY(cudaMallocAsync(&changed, sizeof(int) * size_t(R), ctx->stream));
  int st = mt64_draw(ctx, g, int64_t(P) * spp, 1, u);  // problems.cpp:201-202
  if (!st) {
    const dim3 grid((P + kThreads - 1) / kThreads < 1024 ? (P + kThreads - 1) / kThreads : 1024,
                    R < 65535 ? R : 65535);
    if (dtype == MG_F64) {
      pair_norm_kernel<double><<<R, kThreads, 0, ctx->stream>>>(R, P, (const double*)now,
                                                                (const double*)prev, ssn_out,
                                                                changed);
      minirender_pair_kernel<double><<<grid, kThreads, 0, ctx->stream>>>(
          R, P, spp, exponents, target, u, (const double*)now, (const double*)prev,
          (double*)prop, (double*)diff, ssn_out, changed);
    } else {
      pair_norm_kernel<float><<<R, kThreads, 0, ctx->stream>>>(R, P, (const float*)now,
                                                               (const float*)prev, ssn_out,
                                                               changed);
      minirender_pair_kernel<float><<<grid, kThreads, 0, ctx->stream>>>(
          R, P, spp, exponents, target, u, (const float*)now, (const float*)prev, (float*)prop,
          (float*)diff, ssn_out, changed);
    }
    ctx->launches += 2;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) st = cuda_fail(e, "minirender_pair_kernel");
  }
  cudaFreeAsync(u, ctx->stream);
  cudaFreeAsync(changed, ctx->stream);
  return st;
}

int mg_exprate_sample_pair(mg_ctx* ctx, int32_t R, double target_mean, int32_t n, mg_mt64* g,
                           const double* rate_now, const double* rate_prev, double* prop,
                           double* diff, double* ssn) {
  if (!ctx || !g || !rate_now || !rate_prev || !prop || !diff || !ssn)
    return fail(MG_EINVAL, "mg_exprate_sample_pair: null argument");
  if (n < 2) return fail(MG_EINVAL, "exp-rate: samples_per_iter must be at least 2");
  if (R < 1 || R > g->streams) return fail(MG_EINVAL, "mg_exprate_sample_pair: bad sizes");
  // validate_params before drawing (problems.cpp:56-57, :91-94)
  MG_CUDA_TRY(cudaMemsetAsync(ctx->flag, 0, sizeof(int), ctx->stream));
  domain_check_kernel<<<(R + 255) / 256, 256, 0, ctx->stream>>>(R, rate_now, rate_prev, ctx->flag);
  MG_LAUNCH_CHECK(ctx);
  int flag = 0;
  MG_CUDA_TRY(cudaMemcpyAsync(&flag, ctx->flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (flag) return fail(MG_EDOMAIN, "exp-rate: rate must be positive");
  double* u = nullptr;
  MG_CUDA_TRY(cudaMallocAsync(&u, sizeof(double) * size_t(R) * n, ctx->stream));
  int st = mt64_draw(ctx, g, n, 2, u);  // uniform_pos (problems.cpp:60)
  if (!st) {
    exprate_pair_kernel<<<(R + 127) / 128, 128, 0, ctx->stream>>>(R, n, target_mean, u, rate_now,
                                                                  rate_prev, prop, diff, ssn);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) st = cuda_fail(e, "exprate_pair_kernel");
  }
  cudaFreeAsync(u, ctx->stream);
  return st;
}

int mg_multnoise_sample_pair(mg_ctx* ctx, int32_t R, int32_t d, double sigma, int32_t n,
                             const double* target, mg_mt64* g, const double* now,
                             const double* prev, double* prop, double* diff, double* ssn) {
  if (!ctx || !g || !target || !now || !prev || !prop || !diff || !ssn)
    return fail(MG_EINVAL, "mg_multnoise_sample_pair: null argument");
  if (sigma < 0.0) return fail(MG_EINVAL, "mult-noise: noise amplitude must be >= 0");
  if (n < 1) return fail(MG_EINVAL, "mult-noise: samples_per_iter must be >= 1");
  if (d < 1 || R < 1 || R > g->streams) return fail(MG_EINVAL, "mg_multnoise_sample_pair: bad sizes");
  double* u = nullptr;
  MG_CUDA_TRY(cudaMallocAsync(&u, sizeof(double) * size_t(R) * d * n, ctx->stream));
  int st = mt64_draw(ctx, g, int64_t(d) * n, 1, u);  // problems.cpp:125-126
  if (!st) {
    multnoise_pair_kernel<<<(R + 127) / 128, 128, 0, ctx->stream>>>(R, d, n, sigma, target, u, now,
                                                                    prev, prop, diff, ssn);
    ctx->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) st = cuda_fail(e, "multnoise_pair_kernel");
  }
  cudaFreeAsync(u, ctx->stream);
  return st;
}

}  // extern "C"
