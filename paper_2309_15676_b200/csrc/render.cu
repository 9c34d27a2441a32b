// Fused mini-render iteration: MiniRenderProblem::sample_pair (rows A3/A4,
// problems.cpp:177-217) + the fused meta-estimator update (A8-A11) in ONE
// pass per pixel.  The sample pair never touches HBM: per pixel the kernel
// draws its spp uniforms (from a pre-drawn mt19937_64 buffer — the
// reference's exact stream — or from a Philox4x32-10 counter), evaluates
// the estimator at pi_t and the common-random-number difference against
// pi_{t-1}, and feeds both straight into Moment2 x2 / MetaEstimator / the
// projected update, writing pi_{t+1} over pi_{t-1} (ping-pong) and folding
// the next step norm, #changed and the loss into the last-CTA reduction.
//
// HBM bytes per pixel (fp32, Philox): read b, T, pi_t, pi_{t-1}, m2p, m2d,
// mean, var, alpha = 36 B; write m2p, m2d, mean, var, alpha, pi_{t+1} = 24 B
// -> 60 B/pixel (vs 84 B for sample_pair + mg_meta_update separately).
#include <math.h>

#include "meta_math.cuh"
#include "mg_common.cuh"
#include "philox.cuh"
#include "problems.cuh"
#include "render.cuh"

namespace mg {
bool g_render_vec = true;
bool g_render_fast = true;  // mg_set_option("render_fast", 0): IEEE fp32 kernel everywhere  // mg_set_option("render_vec", 0) forces one pixel per thread
namespace {

constexpr int kThreads = 256;

// Uniforms of one pixel into u[0..spp): Philox in pairs (one 4x32 block
// gives two 53-bit doubles) or the mt19937_64 buffer (pixel-major).
template <int MAXS>
__device__ __forceinline__ void pixel_uniforms(const RenderK& k, int64_t j,
                                               const double* __restrict__ uniforms, double* u) {
  if (k.philox) {
#pragma unroll
    for (int q = 0; q < MAXS; q += 2) {
      if (q < k.spp) {
        const Philox4 r = philox4x32_10(Philox4{{uint32_t(j) + k.pixel_offset, k.iteration,
                                                 uint32_t(q >> 1),
                                                 k.stream}},
                                        uint32_t(k.key), uint32_t(k.key >> 32));
        philox_uniform2(r, u[q], u[q + 1 < MAXS ? q + 1 : q]);
      }
    }
  } else {
    const double* src = uniforms + j * k.spp;  // problems.cpp:201-202
#pragma unroll
    for (int q = 0; q < MAXS; ++q)
      if (q < k.spp) u[q] = src[q];
  }
}

// One pixel: sample pair (problems.cpp:205-213) + fused meta update.
template <class T, bool FIRST, int MAXS>
__device__ __forceinline__ void render_pixel(const RenderK& k, const StepScal& s, bool same,
                                             int64_t j, const double* __restrict__ uniforms,
                                             T bj, T target, T a, T a_prev, T& m2p, T& m2d,
                                             T& mean, T& var, T& ap, T& pout, T& prop, T& diff,
                                             Acc& acc) {
  T cross, mb;
  if (k.spp <= MAXS) {
    double u[MAXS];
    pixel_uniforms<MAXS>(k, j, uniforms, u);
    minirender_terms_arr<T, MAXS>(double(bj), k.spp, u, cross, mb);
  } else if (k.philox) {
    minirender_terms_fn<T>(double(bj), k.spp,
                           [&](int q) {
                             return philox_uniform_at(k.key, uint32_t(j) + k.pixel_offset,
                                                      k.iteration,
                                                      uint32_t(q), k.stream);
                           },
                           cross, mb);
  } else {
    const double* u = uniforms + j * k.spp;
    minirender_terms_fn<T>(double(bj), k.spp, [&](int q) { return u[q]; }, cross, mb);
  }
  prop = (T(2) * a) * cross - (T(2) * target) * mb;      // problems.cpp:205
  diff = same ? T(0) : (T(2) * (a - a_prev)) * cross;   // problems.cpp:206-213
  T dl;
  meta_elem<T, FIRST>(k.meta, s, prop, diff, prop, diff, m2p, m2d, mean, var, ap, a, a_prev,
                      target, true, pout, dl, acc);
}

template <class T, bool FIRST, bool VEC>
__global__ void __launch_bounds__(kThreads, sizeof(T) == 4 ? 3 : 2)
    minirender_meta_kernel(int64_t P, RenderK k, const T* __restrict__ b,
                           const T* __restrict__ tgt, const double* __restrict__ uniforms,
                           const T* __restrict__ pnow, T* __restrict__ pprev_next,
                           T* __restrict__ m2p, T* __restrict__ m2d, T* __restrict__ mean,
                           T* __restrict__ var, T* __restrict__ ap, T* __restrict__ prop_out,
                           T* __restrict__ diff_out, mg_update_scalars* sc,
                           ReducePartials* partials, unsigned int* counter) {
  constexpr int MAXS = 4;
  const StepScal s = load_step_scalars(k.meta, sc);
  const bool same = __ldcg(&sc->changed) == 0.0;  // (params == prev).all(), problems.cpp:206
  Acc acc;
  const int64_t tid = int64_t(blockIdx.x) * kThreads + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * kThreads;
  constexpr int W = VEC ? VecOf<T>::width : 1;
  const int64_t items = VEC ? P / W : 0;
  if constexpr (VEC) {
    for (int64_t it = tid; it < items; it += stride) {
      const int64_t base = it * W;
      const Pack<T> B = ld_stream(b + base), TG = ld_stream(tgt + base);
      const Pack<T> A = ld_plain(pnow + base), AQ = ld_plain(pprev_next + base);
      Pack<T> M2P{}, M2D{}, ME{}, VA{}, AL{}, PO, PR, DF;
      if (!FIRST) {
        M2P = ld_plain(m2p + base);
        ME = ld_plain(mean + base);
        VA = ld_plain(var + base);
        AL = ld_plain(ap + base);
      }
      if (s.cnt0 > 0) M2D = ld_plain(m2d + base);
#pragma unroll
      for (int w = 0; w < W; ++w)
        render_pixel<T, FIRST, MAXS>(k, s, same, base + w, uniforms, B.v[w], TG.v[w], A.v[w],
                                     AQ.v[w], M2P.v[w], M2D.v[w], ME.v[w], VA.v[w], AL.v[w],
                                     PO.v[w], PR.v[w], DF.v[w], acc);
      st_plain(m2p + base, M2P);
      if (s.active) st_plain(m2d + base, M2D);
      st_plain(mean + base, ME);
      st_plain(var + base, VA);
      st_plain(ap + base, AL);
      st_plain(pprev_next + base, PO);
      if (k.record < 0) {
        if (prop_out) st_plain(prop_out + base, PR);
        if (diff_out) st_plain(diff_out + base, DF);
      } else if (k.record >= base && k.record < base + W) {
#pragma unroll
        for (int w = 0; w < W; ++w)
          if (base + w == k.record) {
            if (prop_out) prop_out[0] = PR.v[w];
            if (diff_out) diff_out[0] = DF.v[w];
          }
      }
    }
  }
  for (int64_t j = items * W + tid; j < P; j += stride) {
    T M2P = FIRST ? T(0) : m2p[j];
    T M2D = s.cnt0 > 0 ? m2d[j] : T(0);
    T ME = FIRST ? T(0) : mean[j];
    T VA = FIRST ? T(0) : var[j];
    T AL = FIRST ? T(0) : ap[j];
    T PO, PR, DF;
    render_pixel<T, FIRST, MAXS>(k, s, same, j, uniforms, b[j], tgt[j], pnow[j], pprev_next[j],
                                 M2P, M2D, ME, VA, AL, PO, PR, DF, acc);
    m2p[j] = M2P;
    if (s.active) m2d[j] = M2D;
    mean[j] = ME;
    var[j] = VA;
    ap[j] = AL;
    pprev_next[j] = PO;
    if (k.record < 0) {
      if (prop_out) prop_out[j] = PR;
      if (diff_out) diff_out[j] = DF;
    } else if (j == k.record) {
      if (prop_out) prop_out[0] = PR;
      if (diff_out) diff_out[0] = DF;
    }
  }
  grid_reduce4<kThreads>(acc.partials(), partials, counter, [&](const ReducePartials& t) {
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

template <class T>
int launch(mg_ctx* ctx, int64_t P, const RenderK& k, bool first, const void* b, const void* t,
           const double* u, const void* pnow, void* pprev, void* m2p, void* m2d, void* mean,
           void* var, void* ap, void* prop_out, void* diff_out, mg_update_scalars* sc) {
  // fp32, no per-pixel outputs, large P: the TMA-fed fast kernel
  // (render_fast.cu; Philox, or the exact mt64 draws as a tenth stream)
  if (sizeof(T) == 4 && g_render_fast && k.record < 0 && !prop_out && !diff_out) {
    const int rc = launch_minirender_fast(ctx, P, k, first, (const float*)b, (const float*)t,
                                          (const float*)pnow, (float*)pprev, (float*)m2p,
                                          (float*)m2d, (float*)mean, (float*)var, (float*)ap, sc,
                                          u);
    if (rc != MG_EUNSUPPORTED) return rc;
  }
  // fp32: 4 pixels per thread (16-byte packs, ILP across 4 Philox/pow
  // chains); fp64: one pixel per thread (the packed fp64 body needs 155 regs)
  const bool vec = g_render_vec && sizeof(T) == 4 && aligned16(b) && aligned16(t) && aligned16(pnow) && aligned16(pprev) &&
                   aligned16(m2p) && aligned16(m2d) && aligned16(mean) && aligned16(var) &&
                   aligned16(ap) && (k.record >= 0 || !prop_out || aligned16(prop_out)) &&
                   (k.record >= 0 || !diff_out || aligned16(diff_out));
  const int64_t items = vec ? (P + VecOf<T>::width - 1) / VecOf<T>::width : P;
  const int grid = grid_for(ctx, items, kThreads, 8);
  auto run = [&](auto kernel) {
    kernel<<<grid, kThreads, 0, ctx->stream>>>(
        P, k, (const T*)b, (const T*)t, u, (const T*)pnow, (T*)pprev, (T*)m2p, (T*)m2d, (T*)mean,
        (T*)var, (T*)ap, (T*)prop_out, (T*)diff_out, sc, ctx->partials, ctx->counter);
  };
  if (first)
    vec ? run(minirender_meta_kernel<T, true, true>) : run(minirender_meta_kernel<T, true, false>);
  else
    vec ? run(minirender_meta_kernel<T, false, true>) : run(minirender_meta_kernel<T, false, false>);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

}  // namespace
}  // namespace mg

using namespace mg;

extern "C" int mg_minirender_meta_iteration(mg_ctx* ctx, int32_t dtype, int64_t P,
                                            const mg_render_args* a, const void* exponents,
                                            const void* target, const double* uniforms,
                                            const void* params_now, void* params_prev_next,
                                            void* m2_prop, void* m2_diff, void* mean, void* var,
                                            void* alpha_prev, mg_update_scalars* scalars,
                                            void* prop_out, void* diff_out) {
  MG_NVTX("mg_minirender_meta_iteration");
  if (!ctx || !a || !scalars) return fail(MG_EINVAL, "mg_minirender_meta_iteration: null argument");
  if (P < 1) return fail(MG_EINVAL, "mini-render: pixel_count must be >= 1");
  if (a->spp < 2) return fail(MG_EINVAL, "mini-render: spp must be at least 2");
  if (a->rng_kind == MG_RNG_MT64 && !uniforms)
    return fail(MG_EINVAL, "mg_minirender_meta_iteration: mt64 mode needs the drawn uniforms");
  if (!exponents || !target || !params_now || !params_prev_next || !m2_prop || !m2_diff ||
      !mean || !var || !alpha_prev)
    return fail(MG_EINVAL, "mg_minirender_meta_iteration: null buffer");
  if (a->update.diff_norm != MG_DIFF_NORM_GLOBAL)
    return fail(MG_EUNSUPPORTED, "mg_minirender_meta_iteration: global diff norm only");
  {
    const mg_meta_update_args* u = &a->update;
    if (u->prop_coef_device && !(u->beta_f > 0.0) && !u->prop_pow_advance)
      return fail(MG_EINVAL,
                  "mg_minirender_meta_iteration: prop_coef_device with beta_f = 0 needs prop_pow_advance");
  }
  RenderK k;
  k.meta.lr = a->update.meta.lr;
  k.meta.eps_step = a->update.meta.eps_step;
  k.meta.eps_alpha = a->update.meta.eps_alpha;
  k.meta.clip = a->update.meta.clip_enabled;
  k.meta.prop_coef = a->update.prop_coef;
  k.meta.beta_f = a->update.beta_f;
  k.meta.prop_dev = a->update.prop_coef_device;
  k.meta.prop_adv = a->update.prop_pow_advance;
  k.meta.beta_delta = a->update.beta_delta;
  k.meta.diff_norm = MG_DIFF_NORM_GLOBAL;
  k.meta.project = 1;  // problems.cpp:228: params = params.max(0.0)
  k.meta.proj_lo = 0.0;
  k.meta.proj_hi = 0.0;
  k.meta.ssn_from_host = a->update.ssn_from_host;
  k.meta.ssn_host = a->update.ssn_host;
  k.spp = a->spp;
  k.philox = a->rng_kind == MG_RNG_PHILOX;
  k.key = a->key;
  k.iteration = a->iteration;
  k.stream = a->stream;
  k.pixel_offset = a->pixel_offset;
  k.record = a->record_plus1 > 0 ? int64_t(a->record_plus1) - 1 : -1;
  if (k.record >= P) return fail(MG_EINVAL, "mg_minirender_meta_iteration: record index out of range");
  const bool first = a->update.first_step != 0;
  if (dtype == MG_F32)
    return launch<float>(ctx, P, k, first, exponents, target, uniforms, params_now,
                         params_prev_next, m2_prop, m2_diff, mean, var, alpha_prev, prop_out,
                         diff_out, scalars);
  if (dtype == MG_F64)
    return launch<double>(ctx, P, k, first, exponents, target, uniforms, params_now,
                          params_prev_next, m2_prop, m2_diff, mean, var, alpha_prev, prop_out,
                          diff_out, scalars);
  return fail(MG_EINVAL, "mg_minirender_meta_iteration: unknown dtype");
}
