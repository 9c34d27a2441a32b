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

namespace mg {
namespace {

constexpr int kThreads = 256;

struct RenderK {
  MetaK meta;
  int spp;
  int philox;  // 0: uniforms buffer (mt19937_64 stream), 1: Philox counter
  uint64_t key;
  uint32_t iteration, stream;
};

template <class T, bool FIRST>
__global__ void __launch_bounds__(kThreads)
    minirender_meta_kernel(int64_t P, RenderK k, const T* __restrict__ b,
                           const T* __restrict__ tgt, const double* __restrict__ uniforms,
                           const T* __restrict__ pnow, T* __restrict__ pprev_next,
                           T* __restrict__ m2p, T* __restrict__ m2d, T* __restrict__ mean,
                           T* __restrict__ var, T* __restrict__ ap, T* __restrict__ prop_out,
                           T* __restrict__ diff_out, mg_update_scalars* sc,
                           ReducePartials* partials, unsigned int* counter) {
  const StepScal s = load_step_scalars(k.meta, sc);
  const bool same = __ldcg(&sc->changed) == 0.0;  // (params == prev).all(), problems.cpp:206
  Acc acc;
  for (int64_t j = int64_t(blockIdx.x) * kThreads + threadIdx.x; j < P;
       j += int64_t(gridDim.x) * kThreads) {
    T cross, mb;
    if (k.philox) {
      minirender_terms_fn<T>(double(b[j]), k.spp,
                             [&](int q) {
                               return philox_uniform_at(k.key, uint32_t(j), k.iteration,
                                                        uint32_t(q), k.stream);
                             },
                             cross, mb);
    } else {
      const double* u = uniforms + j * k.spp;  // pixel-major (problems.cpp:201-202)
      minirender_terms_fn<T>(double(b[j]), k.spp, [&](int q) { return u[q]; }, cross, mb);
    }
    const T a = pnow[j];
    const T a_prev = pprev_next[j];
    const T target = tgt[j];
    const T prop = (T(2) * a) * cross - (T(2) * target) * mb;          // :205
    const T diff = same ? T(0) : (T(2) * (a - a_prev)) * cross;       // :206-213
    if (prop_out) prop_out[j] = prop;
    if (diff_out) diff_out[j] = diff;
    T M2P = FIRST ? T(0) : m2p[j];
    T M2D = s.cnt0 > 0 ? m2d[j] : T(0);
    T ME = FIRST ? T(0) : mean[j];
    T VA = FIRST ? T(0) : var[j];
    T AP = FIRST ? T(0) : ap[j];
    T PO, DL;
    meta_elem<T, FIRST>(k.meta, s, prop, diff, prop, diff, M2P, M2D, ME, VA, AP, a, a_prev,
                        target, true, PO, DL, acc);
    m2p[j] = M2P;
    if (s.active) m2d[j] = M2D;
    mean[j] = ME;
    var[j] = VA;
    ap[j] = AP;
    pprev_next[j] = PO;
  }
  grid_reduce4<kThreads>(acc.partials(), partials, counter, [&](const ReducePartials& t) {
    sc->ssn = t.ssn;
    sc->changed = t.changed;
    sc->loss = t.loss;
    sc->nonfinite = t.nonfinite;
    sc->diff_count = s.cnt;
    sc->diff_decay_pow = s.dpow;
    sc->ssn_used = s.ssn;
  });
}

template <class T>
int launch(mg_ctx* ctx, int64_t P, const RenderK& k, bool first, const void* b, const void* t,
           const double* u, const void* pnow, void* pprev, void* m2p, void* m2d, void* mean,
           void* var, void* ap, void* prop_out, void* diff_out, mg_update_scalars* sc) {
  const int grid = grid_for(ctx, P, kThreads, 8);
  auto run = [&](auto kernel) {
    kernel<<<grid, kThreads, 0, ctx->stream>>>(
        P, k, (const T*)b, (const T*)t, u, (const T*)pnow, (T*)pprev, (T*)m2p, (T*)m2d, (T*)mean,
        (T*)var, (T*)ap, (T*)prop_out, (T*)diff_out, sc, ctx->partials, ctx->counter);
  };
  first ? run(minirender_meta_kernel<T, true>) : run(minirender_meta_kernel<T, false>);
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
  RenderK k;
  k.meta.lr = a->update.meta.lr;
  k.meta.eps_step = a->update.meta.eps_step;
  k.meta.eps_alpha = a->update.meta.eps_alpha;
  k.meta.clip = a->update.meta.clip_enabled;
  k.meta.prop_coef = a->update.prop_coef;
  k.meta.beta_delta = a->update.beta_delta;
  k.meta.diff_norm = MG_DIFF_NORM_GLOBAL;
  k.meta.project = 1;  // problems.cpp:228: params = params.max(0.0)
  k.meta.proj_lo = 0.0;
  k.meta.ssn_from_host = a->update.ssn_from_host;
  k.meta.ssn_host = a->update.ssn_host;
  k.spp = a->spp;
  k.philox = a->rng_kind == MG_RNG_PHILOX;
  k.key = a->key;
  k.iteration = a->iteration;
  k.stream = a->stream;
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
