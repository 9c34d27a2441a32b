// F1 slice: path-traced gradient samples for BASELINE.json
// configs[0] — a textured quad lit by a rectangular area light, direct
// lighting only (max depth 1), Lambertian BSDF, RGB albedo texture of R x R
// texels (nearest lookup).  The reference has no renderer;
// scene and estimators are specified in DESIGN.md §F1 and restated on the
// CPU in oracle/metagrad_oracle.c (mgo_quad_*), the oracle for these kernels.
//
// Per pixel, three Philox-addressed samples (counter = pixel, iteration,
// sample id, stream): A and B form the proportional sample with
// decorrelated residual and derivative (r_A * dI_B + r_B * dI_A), C is the
// finite-difference sample evaluated at theta_t and theta_{t-1} on the same
// random numbers (dI_C * (dI_A + dI_B)).  The adjoint scatter into the
// texture uses 2^-40 fixed-point int64 atomics, privatised in shared memory
// for small textures: integer addition is associative, so the gradient is
// bit-identical run to run and to the CPU oracle in fp64.
#include <math.h>

#include "mg_common.cuh"
#include "philox.cuh"

namespace mg {
namespace {

constexpr int kQThreads = 256;
constexpr double kHalf = 1.2, kLX0 = -0.5, kLX1 = 0.5, kLY0 = 0.8, kLY1 = 1.4, kLZ = 1.5;
constexpr double kFix = 1099511627776.0;  // 2^40
constexpr double kPi = 3.14159265358979323846;

struct QuadK {
  int W, H, R;
  int row0, row1;  // image rows [row0, row1) of this tile
  double Le[3];
  uint64_t key;
  uint32_t iteration, stream;
  const uint32_t* it_offset;  // device iteration offset or null (mg_ctx_set_iteration_offset)
};

__device__ __forceinline__ void quad_uniforms(uint64_t key, uint32_t pix, uint32_t it, uint32_t sid,
                                              uint32_t st, double u[4]) {
  const Philox4 r = philox4x32_10(Philox4{{pix, it, sid, st}}, uint32_t(key), uint32_t(key >> 32));
#pragma unroll
  for (int k = 0; k < 4; ++k) u[k] = double(r.x[k]) * 0x1.0p-32;
}

// One NEE sample: texel index (-1: miss) and K_c = Le_c / pi * G * A.
__device__ __forceinline__ int quad_sample(const QuadK& q, int px, int py, const double u[4],
                                           double K[3]) {
  const double nx = ((double(px) + u[0]) / double(q.W)) * 2.0 - 1.0;
  const double ny = 1.0 - ((double(py) + u[1]) / double(q.H)) * 2.0;
  const double x = kHalf * nx, y = kHalf * ny;
  if (x < -1.0 || x > 1.0 || y < -1.0 || y > 1.0) {
    K[0] = K[1] = K[2] = 0.0;
    return -1;
  }
  int tx = int(((x + 1.0) * 0.5) * double(q.R)), ty = int(((y + 1.0) * 0.5) * double(q.R));
  tx = tx > q.R - 1 ? q.R - 1 : tx;
  ty = ty > q.R - 1 ? q.R - 1 : ty;
  const double lx = kLX0 + u[2] * (kLX1 - kLX0);
  const double ly = kLY0 + u[3] * (kLY1 - kLY0);
  const double wx = lx - x, wy = ly - y, wz = kLZ;
  const double d2 = (wx * wx + wy * wy) + wz * wz;
  const double inv = 1.0 / sqrt(d2);
  const double cz = wz * inv;
  const double area = (kLX1 - kLX0) * (kLY1 - kLY0);
  const double G = ((cz * cz) / d2) * area;
#pragma unroll
  for (int c = 0; c < 3; ++c) K[c] = (q.Le[c] / kPi) * G;
  return ty * q.R + tx;
}

template <class T>
__global__ void __launch_bounds__(kQThreads)
    quad_render_kernel(QuadK q, int spp, const T* __restrict__ tex, T* __restrict__ img) {
  const int npix = q.W * q.H;
  const int T_ = q.R * q.R;
  for (int pix = blockIdx.x * kQThreads + threadIdx.x; pix < npix; pix += gridDim.x * kQThreads) {
    const int px = pix % q.W, py = pix / q.W;
    double acc[3] = {0.0, 0.0, 0.0};
    for (int s = 0; s < spp; ++s) {
      double u[4], K[3];
      quad_uniforms(q.key, uint32_t(pix), 0xffffffffu, uint32_t(s), q.stream, u);
      const int t = quad_sample(q, px, py, u, K);
      if (t < 0) continue;
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c] += double(tex[c * T_ + t]) * K[c];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) img[size_t(c) * npix + pix] = T(acc[c] / double(spp));
  }
}

__device__ __forceinline__ long long to_fix(double v) { return llrint(v * kFix); }

// shared-memory accumulator: atomicAdd (ATOMS); global: a RED (red_add_u64)
template <bool SHARED>
__device__ __forceinline__ void acc_add(unsigned long long* p, unsigned long long v) {
  if constexpr (SHARED)
    atomicAdd(p, v);
  else
    red_add_u64(p, v);
}

// SHARED: privatised accumulators [2][3][T] in dynamic shared memory.
template <class T, bool SHARED>
__global__ void __launch_bounds__(kQThreads)
    quad_pair_kernel(QuadK q, const T* __restrict__ target_img, const T* __restrict__ now,
                     const T* __restrict__ prev, unsigned long long* __restrict__ acc_g,
                     ReducePartials* partials, unsigned int* counter, double* loss_out) {
  extern __shared__ unsigned long long acc_s[];
  if (q.it_offset) q.iteration += __ldg(q.it_offset);
  const int npix = q.W * q.H;
  const int T_ = q.R * q.R;
  const int pix0 = q.row0 * q.W, pix1 = q.row1 * q.W;
  unsigned long long* acc = SHARED ? acc_s : acc_g;
  if (SHARED) {
    for (int k = threadIdx.x; k < 6 * T_; k += kQThreads) acc_s[k] = 0ull;
    __syncthreads();
  }
  double loss = 0.0;
  for (int pix = pix0 + blockIdx.x * kQThreads + threadIdx.x; pix < pix1;
       pix += gridDim.x * kQThreads) {
    const int px = pix % q.W, py = pix / q.W;
    double uA[4], uB[4], uC[4], KA[3], KB[3], KC[3];
    quad_uniforms(q.key, uint32_t(pix), q.iteration, 0u, q.stream, uA);
    quad_uniforms(q.key, uint32_t(pix), q.iteration, 1u, q.stream, uB);
    quad_uniforms(q.key, uint32_t(pix), q.iteration, 2u, q.stream, uC);
    const int tA = quad_sample(q, px, py, uA, KA);
    const int tB = quad_sample(q, px, py, uB, KB);
    const int tC = quad_sample(q, px, py, uC, KC);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double Is = double(target_img[size_t(c) * npix + pix]);
      const double rA = (tA >= 0 ? double(now[c * T_ + tA]) * KA[c] : 0.0) - Is;
      const double rB = (tB >= 0 ? double(now[c * T_ + tB]) * KB[c] : 0.0) - Is;
      const double dI =
          tC >= 0 ? (double(now[c * T_ + tC]) - double(prev[c * T_ + tC])) * KC[c] : 0.0;
      loss += rA * rB;
      if (tB >= 0) {
        acc_add<SHARED>(&acc[c * T_ + tB], (unsigned long long)to_fix(rA * KB[c]));
        acc_add<SHARED>(&acc[3 * T_ + c * T_ + tB], (unsigned long long)to_fix(dI * KB[c]));
      }
      if (tA >= 0) {
        acc_add<SHARED>(&acc[c * T_ + tA], (unsigned long long)to_fix(rB * KA[c]));
        acc_add<SHARED>(&acc[3 * T_ + c * T_ + tA], (unsigned long long)to_fix(dI * KA[c]));
      }
    }
  }
  if (SHARED) {
    __syncthreads();
    for (int k = threadIdx.x; k < 6 * T_; k += kQThreads)
      if (acc_s[k]) red_add_u64(&acc_g[k], acc_s[k]);
  }
  Acc a;
  a.ssn = loss;
  grid_reduce4<kQThreads>(a.partials(), partials, counter,
                          [&](const ReducePartials& t) { *loss_out = t.ssn; });
}

template <class T>
__global__ void quad_finalize_kernel(int n, unsigned long long* __restrict__ acc, T* __restrict__ prop,
                                     T* __restrict__ diff) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    prop[k] = T(double((long long)acc[k]) / kFix);
    diff[k] = T(double((long long)acc[n + k]) / kFix);
    acc[k] = 0ull;
    acc[n + k] = 0ull;
  }
}

QuadK make_quad(int W, int H, int R, const double* Le, uint64_t key, uint32_t it, uint32_t st) {
  QuadK q;
  q.W = W;
  q.H = H;
  q.R = R;
  q.row0 = 0;
  q.row1 = H;
  for (int c = 0; c < 3; ++c) q.Le[c] = Le[c];
  q.key = key;
  q.iteration = it;
  q.stream = st;
  q.it_offset = nullptr;
  return q;
}

}  // namespace
}  // namespace mg

using namespace mg;

extern "C" {

int mg_quad_render(mg_ctx* ctx, int32_t dtype, int32_t W, int32_t H, int32_t R, const double* Le,
                   int32_t spp, uint64_t key, uint32_t stream, const void* tex, void* img) {
  if (!ctx || !Le || !tex || !img) return fail(MG_EINVAL, "mg_quad_render: null argument");
  if (W < 1 || H < 1 || R < 1 || spp < 1) return fail(MG_EINVAL, "mg_quad_render: bad sizes");
  const QuadK q = make_quad(W, H, R, Le, key, 0u, stream);
  const int grid = grid_for(ctx, int64_t(W) * H, kQThreads, 8);
  if (dtype == MG_F64)
    quad_render_kernel<double><<<grid, kQThreads, 0, ctx->stream>>>(q, spp, (const double*)tex,
                                                                    (double*)img);
  else if (dtype == MG_F32)
    quad_render_kernel<float><<<grid, kQThreads, 0, ctx->stream>>>(q, spp, (const float*)tex,
                                                                   (float*)img);
  else
    return fail(MG_EINVAL, "mg_quad_render: unknown dtype");
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

int mg_quad_sample_pair(mg_ctx* ctx, int32_t dtype, int32_t W, int32_t H, int32_t R,
                        const double* Le, const void* target_img, const void* now,
                        const void* prev, uint64_t key, uint32_t iteration, uint32_t stream,
                        int32_t row0, int32_t row1, void* accum, void* prop, void* diff,
                        double* loss_out) {
  if (!ctx || !Le || !target_img || !now || !prev || !accum || !prop || !diff || !loss_out)
    return fail(MG_EINVAL, "mg_quad_sample_pair: null argument");
  if (W < 1 || H < 1 || R < 1) return fail(MG_EINVAL, "mg_quad_sample_pair: bad sizes");
  if (row0 < 0 || row1 > H || row0 > row1) return fail(MG_EINVAL, "mg_quad_sample_pair: bad rows");
  QuadK q = make_quad(W, H, R, Le, key, iteration, stream);
  q.row0 = row0;
  q.row1 = row1;
  q.it_offset = ctx->it_offset;
  const int T_ = R * R;
  const size_t smem = sizeof(unsigned long long) * 6 * size_t(T_);
  // shared-memory privatised accumulators when they fit and the tile has
  // enough pixels (>= 16 per accumulator word) to amortise each CTA's
  // zero-fill and flush of 6 R^2 words; below that, global atomics (64^2
  // image / 32^2 texture: 21.7 -> 17.6 us per graph-replayed iteration)
  const bool shared = smem <= 96 * 1024 && int64_t(W) * (row1 - row0) >= 16 * 6 * int64_t(T_);
  const int grid = grid_for(ctx, int64_t(W) * (row1 - row0) + 1, kQThreads, shared ? 2 : 8);
  auto go = [&](auto tag) {
    using T = decltype(tag);
    if (shared) {
      cudaFuncSetAttribute(quad_pair_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(smem));
      quad_pair_kernel<T, true><<<grid, kQThreads, smem, ctx->stream>>>(
          q, (const T*)target_img, (const T*)now, (const T*)prev, (unsigned long long*)accum,
          ctx->partials, ctx->counter, loss_out);
    } else {
      quad_pair_kernel<T, false><<<grid, kQThreads, 0, ctx->stream>>>(
          q, (const T*)target_img, (const T*)now, (const T*)prev, (unsigned long long*)accum,
          ctx->partials, ctx->counter, loss_out);
    }
    quad_finalize_kernel<T><<<grid_for(ctx, 3 * T_, 256, 4), 256, 0, ctx->stream>>>(
        3 * T_, (unsigned long long*)accum, (T*)prop, (T*)diff);
  };
  if (dtype == MG_F64)
    go(double{});
  else if (dtype == MG_F32)
    go(float{});
  else
    return fail(MG_EINVAL, "mg_quad_sample_pair: unknown dtype");
  ctx->launches += 1;
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

}  // extern "C"
