// Fused mini-render iteration, fp32 fast mode (Philox draws): the sample
// pair of MiniRenderProblem::sample_pair (problems.cpp:197-217) and the
// fused meta update (A8-A11, moment2.hpp:30-39, meta.hpp:90-113,
// harness.cpp:144-187) in one pass per pixel, with the nine input streams
// (b, T, pi_t, pi_{t-1}, m2_prop, m2_diff, mean, var, alpha_prev) fed by 1-D
// TMA bulk copies through a shared-memory ring, so the bytes in flight do not
// depend on how long a warp spends in the (long) per-pixel arithmetic.
//
// Numerics: the same expressions as render.cu's IEEE kernel, in fp32 with
// FMA contraction (this translation unit is built with --fmad=true; the fp64
// parity kernels are not in it) and the approximate fp32 division / square
// root / reciprocal (div.full, sqrt.approx, rcp.approx: <= 2 ulp).  The
// fp32 fast mode is judged by tolerance against the fp64 oracle (<= 1e-4,
// DESIGN.md §5); these choices stay ~1e-7 relative per operation.
//
// HBM bytes per pixel: 36 read + 24 written = 60 B (fp32).
#include <math.h>

#include "philox.cuh"
#include "render.cuh"
#include "tma.cuh"

namespace mg {

int g_render_fast_variant = -1;
int render_fast_variants();

namespace {

constexpr int kArrays = 9;  // b, T, now, prev, m2p, m2d, mean, var, ap

struct FastVariant {
  int threads, stages, ctas_per_sm, unit;  // unit: threads per TMA ring
};
// shared memory per SM: ctas x stages x 9 x threads x 16 B (<= 216 KB)
__host__ __device__ constexpr FastVariant fast_variant(int i) {
  return i == 0 ? FastVariant{256, 3, 2, 256}
       : i == 1 ? FastVariant{128, 4, 3, 128}
       : i == 2 ? FastVariant{128, 3, 4, 128}
       : i == 3 ? FastVariant{192, 4, 2, 192}
       : i == 4 ? FastVariant{128, 2, 6, 128}
       : i == 5 ? FastVariant{128, 4, 3, 32}
       : i == 6 ? FastVariant{128, 3, 4, 32}
       : i == 7 ? FastVariant{192, 4, 2, 32}
       : i == 8 ? FastVariant{256, 3, 2, 32}
       : i == 9 ? FastVariant{128, 2, 6, 32}
       : i == 10 ? FastVariant{256, 2, 3, 32}
       : i == 11 ? FastVariant{128, 3, 2, 32}
       : i == 12 ? FastVariant{192, 2, 2, 192}
       : i == 13 ? FastVariant{512, 2, 1, 32}
       : i == 14 ? FastVariant{640, 2, 1, 32}
       : i == 15 ? FastVariant{768, 2, 1, 32}
                 : FastVariant{512, 3, 1, 32};
}
constexpr int kNumFastVariants = 17;
// interleaved sweep at 16.7M pixels (tools/render_fast_sweep.py): spp 2 ->
// per-warp rings in one 512-thread CTA per SM (variant 13: 0.162 ms, 0.95
// of HBM; the 128-256-thread shapes 0.172-0.193 ms); spp >= 3 (more
// arithmetic per byte) -> one ring per 192-thread CTA (variant 3; the wide
// shapes 0.222-0.229 ms against 0.208)
constexpr int default_fast_variant(int spp) { return spp == 2 ? 13 : 3; }
// the exact-stream form moves SPP doubles more per pixel: two 192-thread
// stages (ncu, 16.7M px: 0.197 ms spp 2 / 0.218 ms spp 3 vs IEEE 0.276 / 0.297)
constexpr int default_fast_variant_mt(int) { return 12; }

__device__ __forceinline__ float fdiv(float a, float b) {
  float r;
  asm("div.full.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float frcp(float a) {
  float r;
  asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ float fsqrt(float a) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ float fex2(float a) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ float flg2(float a) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}

// u^b for u in [0, 1), b >= 0 (problems.cpp:187 std::pow on the fast path):
// pow(u, 0) = 1, pow(0, b > 0) = 0 as in libm.
__device__ __forceinline__ float powf01(float u, float b) {
  const float r = fex2(b * flg2(u));
  return b == 0.f ? 1.f : (u == 0.f ? 0.f : r);
}

// Per-launch constants of the step, in fp32 (formed once per thread from
// the fp64 step scalars of load_step_scalars).
struct FastScal {
  float c_prop, c_diff, inv_norm, ssn, eps_alpha, neg_lr, eps_step;
  bool active, has_var_diff, has_m2d, clip, same;
};

// One pixel: sample pair + fused meta update (render.cu render_pixel with
// the fp32 fast operations).  u[] holds the pixel's SPP uniforms.
template <bool FIRST, int SPP>
__device__ __forceinline__ void fast_pixel(const FastScal& f, const float (&u)[SPP], float bj,
                                           float target, float a, float a_prev, float& m2p,
                                           float& m2d, float& mean, float& var, float& ap,
                                           float& pout) {
  // kernel_terms (problems.cpp:177-195), cancellation-free pairwise form
  const float bp1 = bj + 1.f;
  float sum = 0.f, pairs = 0.f;
#pragma unroll
  for (int s = 0; s < SPP; ++s) {
    const float basis = bp1 * powf01(u[s], bj);
    pairs += basis * sum;
    sum += basis;
  }
  constexpr float inv_pairs = 2.f / float(SPP * (SPP - 1));  // exact for SPP = 2
  constexpr float inv_n = 1.f / float(SPP);
  const float cross = pairs * inv_pairs;
  const float mb = sum * inv_n;
  const float prop = (2.f * a) * cross - (2.f * target) * mb;        // problems.cpp:205
  const float diff = f.same ? 0.f : (2.f * (a - a_prev)) * cross;    // problems.cpp:206-213
  // Moment2(beta_f).step(prop)
  const float m2p_old = FIRST ? 0.f : m2p;
  m2p = m2p_old + f.c_prop * (prop * prop - m2p_old);
  // decoupled diff variance, global norm (harness.cpp:152-158)
  float m2d_v = f.has_m2d ? m2d : 0.f;
  if (f.active) {
    const float x = diff * f.inv_norm;
    m2d_v = m2d_v + f.c_diff * (x * x - m2d_v);
  }
  m2d = m2d_v;
  const float var_diff = f.has_var_diff ? m2d_v * f.ssn : 0.f;
  // MetaEstimator::step (meta.hpp:103-112)
  float m = (FIRST ? 0.f : mean) + diff;
  float v = (FIRST ? 0.f : var) + var_diff;
  float al = fdiv(m2p, (m2p + v) + f.eps_alpha);
  if (f.clip) al = std_min(al, FIRST ? 0.f : frcp(2.f - ap));  // a_prev = -inf at the first step
  ap = al;
  const float om = 1.f - al;
  m = al * m + om * prop;
  v = (al * al) * v + (om * om) * m2p;
  mean = m;
  var = v;
  const float delta = fdiv(f.neg_lr * m, fsqrt(v) + f.eps_step);
  pout = std_max(a + delta, 0.f);  // problems.cpp:228 (NaN-faithful max)
}

// SPP uniforms of pixel j: Philox4x32-10 blocks {j, it, q/2, stream}, two
// 53-bit uniforms per block (philox.cuh), rounded to fp32 exactly as
// float(double(a53) * 2^-53).
template <int SPP>
__device__ __forceinline__ void fast_uniforms(const RenderK& k, uint32_t j, float (&u)[SPP]) {
#pragma unroll
  for (int q = 0; q < SPP; q += 2) {
    const Philox4 r = philox4x32_10(Philox4{{j, k.iteration, uint32_t(q >> 1), k.stream}},
                                    uint32_t(k.key), uint32_t(k.key >> 32));
    const uint64_t a = (uint64_t(r.x[0]) << 21) ^ uint64_t(r.x[1] >> 11);
    u[q] = __ull2float_rn(a) * 0x1.0p-53f;
    if (q + 1 < SPP) {
      const uint64_t b = (uint64_t(r.x[2]) << 21) ^ uint64_t(r.x[3] >> 11);
      u[q + 1] = __ull2float_rn(b) * 0x1.0p-53f;
    }
  }
}

struct PixAcc {  // per-thread partial sums of one tile (fp32), folded into Acc
  float ssn = 0.f, loss = 0.f;
  unsigned int changed = 0, nonfinite = 0;
  __device__ __forceinline__ void add(float p, float pin, float target) {
    const float d = p - pin;
    ssn += d * d;
    changed += p != pin ? 1u : 0u;
    const float e = p - target;
    loss += e * e;
    nonfinite += isfinite(p) ? 0u : 1u;
  }
  __device__ __forceinline__ void fold(Acc& acc) const {
    acc.ssn += double(ssn);
    acc.loss += double(loss);
    acc.changed += changed;
    acc.nonfinite += nonfinite;
  }
};

// UNIT = THREADS: one ring per CTA (thread 0 issues, __syncthreads between
// consume and refill).  UNIT = 32: one ring per warp (lane 0 issues,
// __syncwarp), so no warp ever waits for another CTA-mate.
// Per-stage shared bytes of one ring: the nine fp32 arrays, and with MT the
// tile's SPP pre-drawn doubles per pixel (the reference's mt19937_64 stream)
template <int TILE, int SPP, bool MT>
__host__ __device__ constexpr int stage_bytes() {
  return kArrays * TILE * int(sizeof(float)) + (MT ? TILE * SPP * int(sizeof(double)) : 0);
}

// MT: the draws are the replicate's exact std::mt19937_64 stream, pre-drawn
// pixel-major (problems.cpp:201-202) and streamed as a tenth TMA array;
// otherwise Philox in registers.
template <bool FIRST, int SPP, int THREADS, int STAGES, int CTAS, int UNIT, bool MT = false>
__global__ void __launch_bounds__(THREADS, CTAS)
    minirender_fast_kernel(int64_t P, RenderK k, const float* __restrict__ b,
                           const float* __restrict__ tgt, const float* __restrict__ pnow,
                           float* __restrict__ pprev_next, float* __restrict__ m2p,
                           float* __restrict__ m2d, float* __restrict__ mean,
                           float* __restrict__ var, float* __restrict__ ap,
                           mg_update_scalars* sc, ReducePartials* partials,
                           unsigned int* counter, const double* __restrict__ uni) {
  static_assert(UNIT == THREADS || UNIT == 32, "one ring per CTA or per warp");
  constexpr int UNITS = THREADS / UNIT;  // rings per CTA
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_all[UNITS * STAGES];
  constexpr int W = 4;
  constexpr int TILE = UNIT * W;
  constexpr int SB = stage_bytes<TILE, SPP, MT>();
  const int unit = threadIdx.x / UNIT, r = threadIdx.x % UNIT;
  uint64_t* full = full_all + unit * STAGES;
  unsigned char* ubase = smem_raw + size_t(unit) * STAGES * SB;
  auto stage_f = [&](int st) { return reinterpret_cast<float*>(ubase + size_t(st) * SB); };
  auto stage_u = [&](int st) {
    return reinterpret_cast<double*>(ubase + size_t(st) * SB + kArrays * TILE * sizeof(float));
  };
  auto unit_sync = [] {
    if constexpr (UNIT == 32) __syncwarp(); else __syncthreads();
  };

  const StepScal s = load_step_scalars(k.meta, sc);
  FastScal f;
  f.c_prop = float(s.c_prop);
  f.c_diff = float(s.c_diff);
  f.inv_norm = float(1.0 / s.norm);
  f.ssn = float(s.ssn);
  f.eps_alpha = float(k.meta.eps_alpha);
  f.neg_lr = float(-k.meta.lr);
  f.eps_step = float(k.meta.eps_step);
  f.active = s.active;
  f.has_var_diff = s.cnt > 0;
  f.has_m2d = s.cnt0 > 0;
  f.clip = k.meta.clip != 0;
  f.same = __ldcg(&sc->changed) == 0.0;  // (params == prev).all(), problems.cpp:206

  const float* src[kArrays] = {b, tgt, pnow, pprev_next, m2p, m2d, mean, var, ap};
  const bool use[kArrays] = {true, true, true, true, !FIRST, f.has_m2d, !FIRST, !FIRST, !FIRST};
  uint32_t tx = 0;
#pragma unroll
  for (int a = 0; a < kArrays; ++a) tx += use[a] ? uint32_t(TILE * sizeof(float)) : 0u;
  if (MT) tx += uint32_t(TILE * SPP * sizeof(double));

  const int64_t tiles = P / TILE;
  const int64_t gunit = int64_t(blockIdx.x) * UNITS + unit, nunits = int64_t(gridDim.x) * UNITS;
  const int64_t my_tiles = gunit < tiles ? (tiles - gunit + nunits - 1) / nunits : 0;
  if (r == 0) {
    for (int st = 0; st < STAGES; ++st) mbar_init(&full[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = l2_evict_first_policy();
  auto issue = [&](int64_t li) {  // r == 0 only
    const int st = int(li % STAGES);
    const int64_t tile = gunit + li * nunits;
    MG_DCHECK((tile + 1) * TILE <= P && st < STAGES);
    mbar_arrive_expect_tx(&full[st], tx);
#pragma unroll
    for (int a = 0; a < kArrays; ++a)
      if (use[a])
        bulk_g2s_hint(stage_f(st) + a * TILE, src[a] + tile * TILE,
                      uint32_t(TILE * sizeof(float)), &full[st], pol);
    if (MT)
      bulk_g2s_hint(stage_u(st), uni + tile * TILE * SPP, uint32_t(TILE * SPP * sizeof(double)),
                    &full[st], pol);
  };
  if (r == 0)
    for (int64_t li = 0; li < my_tiles && li < STAGES; ++li) issue(li);

  Acc acc;
  const int e = r * W;
  for (int64_t li = 0; li < my_tiles; ++li) {
    const int st = int(li % STAGES);
    const int64_t base = (gunit + li * nunits) * TILE + e;
    // Philox draws do not depend on the tile's data: form them before waiting
    float u[W][SPP];
    if constexpr (!MT) {
#pragma unroll
      for (int w = 0; w < W; ++w)
        fast_uniforms<SPP>(k, uint32_t(base + w) + k.pixel_offset, u[w]);
    }
    mbar_wait(&full[st], uint32_t((li / STAGES) & 1));
    if constexpr (MT) {  // float(u) of the drawn doubles, as the IEEE kernel rounds them
      const double* su = stage_u(st) + e * SPP;
#pragma unroll
      for (int w = 0; w < W; ++w)
#pragma unroll
        for (int q = 0; q < SPP; ++q) u[w][q] = float(su[w * SPP + q]);
    }
    const float* sb = stage_f(st) + e;
    const Pack<float> B = ld_plain(sb + 0 * TILE), TG = ld_plain(sb + 1 * TILE);
    const Pack<float> A = ld_plain(sb + 2 * TILE), AQ = ld_plain(sb + 3 * TILE);
    Pack<float> M2P{}, M2D{}, ME{}, VA{}, AL{}, PO;
    if (!FIRST) {
      M2P = ld_plain(sb + 4 * TILE);
      ME = ld_plain(sb + 6 * TILE);
      VA = ld_plain(sb + 7 * TILE);
      AL = ld_plain(sb + 8 * TILE);
    }
    if (f.has_m2d) M2D = ld_plain(sb + 5 * TILE);
    unit_sync();  // every thread of the unit holds stage st in registers: refill it
    if (r == 0 && li + STAGES < my_tiles) {
      fence_proxy_async_smem();
      issue(li + STAGES);
    }
    PixAcc pa;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      fast_pixel<FIRST, SPP>(f, u[w], B.v[w], TG.v[w], A.v[w], AQ.v[w], M2P.v[w], M2D.v[w],
                             ME.v[w], VA.v[w], AL.v[w], PO.v[w]);
      pa.add(PO.v[w], A.v[w], TG.v[w]);
    }
    pa.fold(acc);
    st_stream(m2p + base, M2P);
    if (f.active) st_stream(m2d + base, M2D);
    st_stream(mean + base, ME);
    st_stream(var + base, VA);
    st_stream(ap + base, AL);
    st_stream(pprev_next + base, PO);
  }
  // tail pixels [tiles*TILE, P)
  const int64_t tid = int64_t(blockIdx.x) * THREADS + threadIdx.x;
  for (int64_t j = tiles * TILE + tid; j < P; j += int64_t(gridDim.x) * THREADS) {
    float u[SPP];
    if constexpr (MT) {
#pragma unroll
      for (int q = 0; q < SPP; ++q) u[q] = float(uni[j * SPP + q]);
    } else {
      fast_uniforms<SPP>(k, uint32_t(j) + k.pixel_offset, u);
    }
    float M2P = FIRST ? 0.f : m2p[j];
    float M2D = f.has_m2d ? m2d[j] : 0.f;
    float ME = FIRST ? 0.f : mean[j];
    float VA = FIRST ? 0.f : var[j];
    float AL = FIRST ? 0.f : ap[j];
    const float A = pnow[j], TG = tgt[j];
    float PO;
    fast_pixel<FIRST, SPP>(f, u, b[j], TG, A, pprev_next[j], M2P, M2D, ME, VA, AL, PO);
    PixAcc pa;
    pa.add(PO, A, TG);
    pa.fold(acc);
    m2p[j] = M2P;
    if (f.active) m2d[j] = M2D;
    mean[j] = ME;
    var[j] = VA;
    ap[j] = AL;
    pprev_next[j] = PO;
  }
  grid_reduce4<THREADS>(acc.partials(), partials, counter, [&](const ReducePartials& t) {
    sc->ssn = t.ssn;
    sc->changed = t.changed;
    sc->loss = t.loss;
    sc->nonfinite = t.nonfinite;
    sc->diff_count = s.cnt;
    sc->diff_decay_pow = s.dpow;
    sc->prop_decay_pow = s.ppow;
    sc->ssn_used = s.ssn;
  });
}

template <int V, bool FIRST, int SPP, bool MT>
int run_fast(mg_ctx* ctx, int64_t P, const RenderK& k, const float* b, const float* t,
             const float* pnow, float* pprev, float* m2p, float* m2d, float* mean, float* var,
             float* ap, mg_update_scalars* sc, const double* uni) {
  constexpr FastVariant v = fast_variant(V);
  constexpr int TILE = v.threads * 4;  // pixels per CTA per stage
  constexpr size_t smem = size_t(v.stages) * (v.threads / v.unit) *
                          stage_bytes<v.unit * 4, SPP, MT>();
  auto kernel =
      minirender_fast_kernel<FIRST, SPP, v.threads, v.stages, v.ctas_per_sm, v.unit, MT>;
  if (smem > size_t(227) * 1024) return MG_EUNSUPPORTED;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const int64_t tiles = P / TILE;
  const int fit = int(size_t(227) * 1024 / (smem + 1024));  // CTAs per SM by shared memory
  const int per_sm = v.ctas_per_sm < fit ? v.ctas_per_sm : (fit > 0 ? fit : 1);
  const int64_t want = int64_t(ctx->sm_count) * per_sm;
  int grid = int(tiles < want ? tiles : want);
  if (grid > kMaxReduceBlocks) grid = kMaxReduceBlocks;
  kernel<<<grid, v.threads, smem, ctx->stream>>>(P, k, b, t, pnow, pprev, m2p, m2d, mean, var,
                                                 ap, sc, ctx->partials, ctx->counter, uni);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

template <int V>
int pick_spp(mg_ctx* ctx, int64_t P, const RenderK& k, bool first, const float* b,
             const float* t, const float* pnow, float* pprev, float* m2p, float* m2d,
             float* mean, float* var, float* ap, mg_update_scalars* sc, const double* uni) {
#define MG_FAST_CASE(S)                                                                        \
  case S:                                                                                      \
    if (uni)                                                                                   \
      return first ? run_fast<V, true, S, true>(ctx, P, k, b, t, pnow, pprev, m2p, m2d, mean,  \
                                                var, ap, sc, uni)                              \
                   : run_fast<V, false, S, true>(ctx, P, k, b, t, pnow, pprev, m2p, m2d, mean, \
                                                 var, ap, sc, uni);                            \
    return first ? run_fast<V, true, S, false>(ctx, P, k, b, t, pnow, pprev, m2p, m2d, mean,   \
                                               var, ap, sc, nullptr)                           \
                 : run_fast<V, false, S, false>(ctx, P, k, b, t, pnow, pprev, m2p, m2d, mean,  \
                                                var, ap, sc, nullptr);
  switch (k.spp) {
    MG_FAST_CASE(2)
    MG_FAST_CASE(3)
    MG_FAST_CASE(4)
    default:
      return MG_EUNSUPPORTED;
  }
#undef MG_FAST_CASE
}

}  // namespace

int render_fast_variants() { return kNumFastVariants; }

int launch_minirender_fast(mg_ctx* ctx, int64_t P, const RenderK& k, bool first, const float* b,
                           const float* tgt, const float* pnow, float* pprev_next, float* m2p,
                           float* m2d, float* mean, float* var, float* ap,
                           mg_update_scalars* sc, const double* uniforms) {
  if (k.spp < 2 || k.spp > 4) return MG_EUNSUPPORTED;
  const double* uni = k.philox ? nullptr : uniforms;
  if (!k.philox && !(uniforms && aligned16(uniforms))) return MG_EUNSUPPORTED;
  if (!(aligned16(b) && aligned16(tgt) && aligned16(pnow) && aligned16(pprev_next) &&
        aligned16(m2p) && aligned16(m2d) && aligned16(mean) && aligned16(var) && aligned16(ap)))
    return MG_EUNSUPPORTED;
  const int v = g_render_fast_variant >= 0 ? g_render_fast_variant
                                          : (uni ? default_fast_variant_mt(k.spp)
                                                 : default_fast_variant(k.spp));
  // at least one full 256x4 tile per SM, else the IEEE kernel
  if (P < int64_t(1024) * ctx->sm_count) return MG_EUNSUPPORTED;
  switch (v) {
#define MG_FAST_V(V) \
  case V: return pick_spp<V>(ctx, P, k, first, b, tgt, pnow, pprev_next, m2p, m2d, mean, var, ap, sc, uni);
    MG_FAST_V(0) MG_FAST_V(1) MG_FAST_V(2) MG_FAST_V(3) MG_FAST_V(4)
    MG_FAST_V(5) MG_FAST_V(6) MG_FAST_V(7) MG_FAST_V(8) MG_FAST_V(9) MG_FAST_V(10)
    MG_FAST_V(11) MG_FAST_V(12) MG_FAST_V(13) MG_FAST_V(14) MG_FAST_V(15) MG_FAST_V(16)
#undef MG_FAST_V
    default: return MG_EINVAL;
  }
}

}  // namespace mg
