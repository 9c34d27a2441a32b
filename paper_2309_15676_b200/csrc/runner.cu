// Device-resident run_single / run_experiment (rows A13, A14).
//
// The reference runs each replicate's loop (harness.cpp:90-200) on a
// std::thread pool (harness.cpp:249-272).  Here every replicate is one CTA of
// a single persistent kernel that executes the WHOLE optimisation loop on the
// device: its mt19937_64 stream lives in shared memory, its state vectors in
// global memory (L2-resident at reference sizes), and each iteration is
//   draws -> sample_pair -> Moment2 x2 -> MetaEstimator/Adam -> record -> update
// with no host round trip.  Reductions over a replicate's vector (step norm,
// loss, parameter error) are sequential for dim <= kSeqReduceMax, so in fp64
// the trajectories are bit-identical to the reference's wherever the
// transcendental functions agree.  Mini-render runs go
// through pow, so their parity is tolerance-based anyway; they use the
// fixed block tree at every size (one sequential thread over 4096 values
// per sum was the runner's bottleneck for the S1 configuration).
//
// Recording keeps the reference's extractor series for one coordinate plus
// scalars (harness.cpp:204-244), not full vectors (O(iterations * dim)).
#include <math.h>

#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "mg_common.cuh"
#include "mt64.cuh"
#include "problems.cuh"

namespace mg {
// mg_set_option("cluster_runner", 0): few-replicate mini-render runs on the
// one-CTA-per-replicate kernel too
bool g_cluster_runner = true;
namespace {

// threads of the one-CTA-per-replicate runner.  S1 shape by replicate count
// (tools/runner_reps_probe.py, run_experiment wall): 256 threads 23.5 / 33.5 /
// 76.6 ms at 148 / 296 / 592 replicates, 512 threads 19.7 / 40.5 / 85.0,
// 1024 threads 19.5 / 39.1 / 77.1 - the device saturates near 1.5-1.8M
// replicate-iterations/s (fp64 pow) either way; 256 keeps 2-3 CTAs per SM.
#ifndef MG_RUN_THREADS
#define MG_RUN_THREADS 256
#endif
constexpr int kThreads = MG_RUN_THREADS;
constexpr int kNumSeries = 11;

template <class T>
struct RunK {
  mg_experiment_config cfg;
  int dim;
  int64_t D;  // draws per sample_pair
  int rep_begin;
  int R;
  const double* truth;      // [dim]
  const double* init;       // [dim]
  const double* exponents;  // [dim] mini-render
  const double* sched;      // [(iterations+1)][dim] or null
  // per-replicate state [R][dim]
  T *params, *prev, *prop, *diff, *iprop, *idiff, *m2p, *m2d, *mean, *var, *ap, *am, *av, *delta,
      *mest, *vest;
  double* ubuf;  // [R][D]
  mg_run_record* recs;
  double* series[kNumSeries];  // [R][iterations] each, or null
  double* final_params;        // [R][dim] or null
  // full per-iteration vectors (harness.hpp:79-88), [R][iterations][8][dim]:
  // params, prop, diff, mean_est, var_est, alpha, delta, true_grad; or null
  double* full;
};

// Up to three independent sums over j in [0, n) of f(j) (returns in
// out[0..2], valid in every thread after the call).  Sequential (one thread
// per sum, index order) for n <= kSeqReduceMax, fixed tree otherwise.
template <class F>
__device__ void block_sums3(int n, F f, double* out, double* sw, bool seq = true) {
  __shared__ double res[3];
  if (seq && n <= kSeqReduceMax) {
    const int t = threadIdx.x;
    if (t == 0 || t == 32 || t == 64) {
      const int which = t / 32;
      double s = 0.0;
      for (int j = 0; j < n; ++j) s += f(j, which);
      res[which] = s;
    }
  } else {
    for (int which = 0; which < 3; ++which) {
      double s = 0.0;
      for (int j = threadIdx.x; j < n; j += kThreads) s += f(j, which);
      s = block_sum<kThreads>(s, sw);
      if (threadIdx.x == 0) res[which] = s;
    }
  }
  __syncthreads();
  out[0] = res[0];
  out[1] = res[1];
  out[2] = res[2];
  __syncthreads();
}

// One sample_pair of the configured problem for this CTA's replicate.
// Returns false on std::domain_error (exp-rate non-positive rate).
template <class T>
__device__ bool sample_pair(const RunK<T>& k, MtBlock& eng, const T* now, const T* prev, bool same,
                            T* prop, T* diff, double* u, double& ssn, double* sw) {
  const mg_experiment_config& c = k.cfg;
  const int d = k.dim;
  if (c.problem == MG_EXP_RATE) {
    // validate_params (problems.cpp:56-57, :91-94) before drawing
    if (!(double(now[0]) > 0.0) || !(double(prev[0]) > 0.0)) return false;
    mt_block_generate(eng, k.D, [&](int64_t i, uint64_t raw) { u[i] = 1.0 - mt_uniform(raw); });
    __shared__ double s_out[3];
    if (threadIdx.x == 0) {
      double sum_c = 0.0, sum_c_sq = 0.0;
      exprate_sums(u, c.samples_per_iter, sum_c, sum_c_sq);
      const double rn = double(now[0]), rp = double(prev[0]);
      const double g = exprate_gradient(c.target_mean, c.samples_per_iter, rn, sum_c, sum_c_sq);
      s_out[0] = g;
      if (rn == rp) {
        s_out[1] = 0.0;
        s_out[2] = 0.0;
      } else {
        s_out[1] = g - exprate_gradient(c.target_mean, c.samples_per_iter, rp, sum_c, sum_c_sq);
        s_out[2] = (rn - rp) * (rn - rp);
      }
      prop[0] = T(s_out[0]);
      diff[0] = T(s_out[1]);
    }
    __syncthreads();
    ssn = s_out[2];
    __syncthreads();
    return true;
  }
  mt_block_generate(eng, k.D, [&](int64_t i, uint64_t raw) { u[i] = mt_uniform(raw); });
  for (int j = threadIdx.x; j < d; j += kThreads) {
    if (c.problem == MG_MULT_NOISE) {
      const double f = multnoise_factor(u, d, c.samples_per_iter, j, c.sigma);
      prop[j] = T((double(now[j]) - k.truth[j]) * f);
      diff[j] = same ? T(0) : T((double(now[j]) - double(prev[j])) * f);
    } else {
      T cross, mb;
      minirender_terms<T>(k.exponents[j], u + size_t(j) * c.spp, c.spp, cross, mb);
      const T a = now[j];
      prop[j] = (T(2) * a) * cross - (T(2) * T(k.truth[j])) * mb;
      diff[j] = same ? T(0) : (T(2) * (a - prev[j])) * cross;
    }
  }
  if (same) {
    ssn = 0.0;
    __syncthreads();
  } else {
    double r[3];
    block_sums3(d, [&](int j, int) {
      const double dd = double(now[j]) - double(prev[j]);
      return dd * dd;
    }, r, sw, c.problem != MG_MINI_RENDER);
    ssn = r[0];
  }
  return true;
}

template <class T>
__global__ void __launch_bounds__(kThreads) run_kernel(RunK<T> k) {
  __shared__ uint64_t mtbuf[2][kMtN];
  __shared__ double sw[kThreads / 32];
  const int r = blockIdx.x;
  const mg_experiment_config& c = k.cfg;
  const int d = k.dim;
  const int iters = c.iterations;
  const size_t off = size_t(r) * d;
  T* params = k.params + off;
  T* prev = k.prev + off;
  T* prop = k.prop + off;
  T* diff = k.diff + off;
  T* iprop = k.iprop + off;
  T* idiff = k.idiff + off;
  T* m2p = k.m2p + off;
  T* m2d = k.m2d + off;
  T* mean = k.mean + off;
  T* var = k.var + off;
  T* ap = k.ap + off;
  T* am = k.am + off;
  T* av = k.av + off;
  T* delta = k.delta + off;
  T* mest = k.mest + off;
  T* vest = k.vest + off;
  double* u = k.ubuf + size_t(r) * k.D;

  // Rng::stream(seed, replicate) (rng.hpp:23-25), seeded in shared memory
  MtBlock eng{{mtbuf[0], mtbuf[1]}, 0, kMtN};
  if (threadIdx.x == 0) {
    const uint64_t rep = uint64_t(k.rep_begin + r);
    mt_seed(mtbuf[0], mg_mix64_dev(mg_mix64_dev(c.seed) ^ (rep + 0x51ed2701e35f3a6dULL)));
  }
  const bool scripted = c.trajectory != MG_TRAJ_OPTIMISE;
  const bool use_meta = c.optimizer == MG_OPT_META;
  for (int j = threadIdx.x; j < d; j += kThreads) {
    const T p0 = T(scripted ? k.sched[j] : k.init[j]);
    params[j] = p0;
    prev[j] = p0;
  }
  __syncthreads();

  double pf_pow = 1.0, pd_pow = 1.0, b1p = 1.0, b2p = 1.0;
  int64_t pf_cnt = 0, pd_cnt = 0, t_adam = 0;
  bool meta_first = true;
  int status = 0, iters_run = 0;
  int64_t draws = 0, evals = 0;
  const int coord = c.coord;

  for (int i = 0; i < iters; ++i) {
    // harness.cpp:116-119
    bool finite = true;
    for (int j = threadIdx.x; j < d; j += kThreads) finite &= isfinite(double(params[j]));
    if (!__syncthreads_and(finite)) {
      status = 2;
      break;
    }
    bool eq = true;
    for (int j = threadIdx.x; j < d; j += kThreads) eq &= (params[j] == prev[j]);
    const bool same_pp = __syncthreads_and(eq);
    const T* sample_prev = use_meta ? prev : params;
    const bool same = use_meta ? same_pp : true;
    double ssn = 0.0;
    if (!sample_pair(k, eng, params, sample_prev, same, prop, diff, u, ssn, sw)) {  // :125-128
      status = 2;
      break;
    }
    const bool two_point = use_meta && !same_pp;  // :129
    draws += k.D;
    evals += k.D * (two_point ? 2 : 1);
    if (use_meta) {
      const T* vp = prop;
      const T* vd = diff;
      double vssn = ssn;
      if (c.independent_variance_samples) {  // :137-142
        if (!sample_pair(k, eng, params, prev, same, iprop, idiff, u, vssn, sw)) {
          status = 2;
          break;
        }
        draws += k.D;
        evals += k.D * (two_point ? 2 : 1);
        vp = iprop;
        vd = idiff;
      }
      // Moment2 scalars (moment2.hpp:34-38), uniform across the block
      const bool pf_first = pf_cnt == 0;
      pf_cnt += 1;
      pf_pow = pf_pow * c.beta_f;
      const double cp = (1.0 - c.beta_f) / (1.0 - pf_pow);
      const bool active = vssn > 0.0;
      const bool pd_had = pd_cnt > 0;
      if (active) {
        pd_cnt += 1;
        pd_pow = pd_pow * c.beta_delta;
      }
      const double cd = (1.0 - c.beta_delta) / (1.0 - pd_pow);
      const double norm = sqrt(vssn);
      const bool per_param = c.diff_norm == MG_DIFF_NORM_PER_PARAM;
      for (int j = threadIdx.x; j < d; j += kThreads) {
        const T x = vp[j];
        const T m2p_old = pf_first ? T(0) : m2p[j];
        const T m2pv = m2p_old + T(cp) * (x * x - m2p_old);  // :144
        m2p[j] = m2pv;
        T m2dv = pd_had ? m2d[j] : T(0);
        T var_diff = T(0);
        if (per_param) {  // :146-151
          const T cs = fabs(params[j] - prev[j]);
          if (active) {
            const T tiny = sizeof(T) == 8 ? T(1e-150) : T(1e-37);
            const T xd = vd[j] / std_max(cs, tiny);
            m2dv = m2dv + T(cd) * (xd * xd - m2dv);
            m2d[j] = m2dv;
          }
          if (pd_cnt > 0) var_diff = m2dv * (cs * cs);
        } else {  // :153-157
          if (active) {
            const T xd = vd[j] / T(norm);
            m2dv = m2dv + T(cd) * (xd * xd - m2dv);
            m2d[j] = m2dv;
          }
          if (pd_cnt > 0) var_diff = m2dv * T(ssn);
        }
        // MetaEstimator::step (meta.hpp:92-112)
        T m = (meta_first ? T(0) : mean[j]) + diff[j];
        T v = (meta_first ? T(0) : var[j]) + var_diff;
        const T a_prev = meta_first ? T(-INFINITY) : ap[j];
        T al = m2pv / ((m2pv + v) + T(c.eps_alpha));
        if (!c.no_alpha_clip) al = std_min(al, T(1) / (T(2) - a_prev));
        ap[j] = al;
        const T om = T(1) - al;
        m = al * m + om * prop[j];
        v = (al * al) * v + (om * om) * m2pv;
        mean[j] = m;
        var[j] = v;
        mest[j] = m;
        vest[j] = v;
        delta[j] = (T(-c.lr) * m) / (sqrt(v) + T(c.eps_step));
      }
      meta_first = false;
    } else {  // Adam (adam.hpp:23-37), harness.cpp:165-167
      const bool first = t_adam == 0;
      t_adam += 1;
      b1p = b1p * c.beta1;
      b2p = b2p * c.beta2;
      const T c1 = T(1.0 - c.beta1), c2 = T(1.0 - c.beta2);
      const T d1 = T(1.0 - b1p), d2 = T(1.0 - b2p);
      for (int j = threadIdx.x; j < d; j += kThreads) {
        const T g = prop[j];
        const T mm = T(c.beta1) * (first ? T(0) : am[j]) + c1 * g;
        const T vv = T(c.beta2) * (first ? T(0) : av[j]) + c2 * (g * g);
        am[j] = mm;
        av[j] = vv;
        const T mh = mm / d1, vh = vv / d2;
        mest[j] = mh;  // adam.hpp:42-43
        vest[j] = vh;
        delta[j] = (T(-c.lr) * mh) / (sqrt(vh) + T(c.adam_eps));
      }
    }
    __syncthreads();
    // record iteration i (harness.cpp:170-180) for coordinate `coord`
    double sums[3];
    // loss (problems.cpp:225) and param_err (harness.cpp:212-215) share
    // the sum of (params - truth)^2, taken in index order.
    block_sums3(d, [&](int j, int) {
      const double e = double(params[j]) - k.truth[j];
      return e * e;
    }, sums, sw, c.problem != MG_MINI_RENDER);
    if (threadIdx.x == 0) {
      const size_t at = size_t(r) * iters + i;
      double loss;
      if (c.problem == MG_EXP_RATE) {
        const double err = 1.0 / double(params[0]) - c.target_mean;  // problems.cpp:84-87
        loss = err * err;
      } else if (c.problem == MG_MULT_NOISE) {
        loss = 0.5 * sums[0];  // problems.cpp:146-149
      } else {
        loss = sums[0];  // problems.cpp:223-226
      }
      double tg;
      const double x = double(params[coord]);
      if (c.problem == MG_EXP_RATE)
        tg = (2.0 * (1.0 / x - c.target_mean)) * (-1.0 / (x * x));  // :78-82
      else if (c.problem == MG_MULT_NOISE)
        tg = x - k.truth[coord];  // :141-144
      else
        tg = 2.0 * (x - k.truth[coord]);  // :219-222
      const double vals[kNumSeries] = {sqrt(sums[0]), loss, double(prop[coord]),
                                       double(diff[coord]), double(mest[coord]),
                                       double(vest[coord]),
                                       use_meta ? double(ap[coord]) : nan(""),
                                       double(delta[coord]), tg, ssn, x};
      for (int s = 0; s < kNumSeries; ++s)
        if (k.series[s]) k.series[s][at] = vals[s];
    }
    if (k.full) {  // RunRecord vectors, harness.cpp:170-179
      double* fr = k.full + (size_t(r) * iters + i) * 8 * size_t(d);
      for (int j = threadIdx.x; j < d; j += kThreads) {
        const double x = double(params[j]);
        double tgj;
        if (c.problem == MG_EXP_RATE)
          tgj = (2.0 * (1.0 / x - c.target_mean)) * (-1.0 / (x * x));
        else if (c.problem == MG_MULT_NOISE)
          tgj = x - k.truth[j];
        else
          tgj = 2.0 * (x - k.truth[j]);
        fr[j] = x;
        fr[size_t(d) + j] = double(prop[j]);
        fr[2 * size_t(d) + j] = double(diff[j]);
        fr[3 * size_t(d) + j] = double(mest[j]);
        fr[4 * size_t(d) + j] = double(vest[j]);
        fr[5 * size_t(d) + j] = use_meta ? double(ap[j]) : nan("");
        fr[6 * size_t(d) + j] = double(delta[j]);
        fr[7 * size_t(d) + j] = tgj;
      }
    }
    iters_run = i + 1;
    // prev = params; params += delta; project (harness.cpp:182-188)
    for (int j = threadIdx.x; j < d; j += kThreads) {
      const T p = params[j];
      prev[j] = p;
      T np;
      if (scripted) {
        np = T(k.sched[size_t(i + 1) * d + j]);
      } else {
        np = p + delta[j];
        if (c.problem == MG_EXP_RATE)
          np = std_max(np, T(1e-4));  // problems.cpp:89
        else if (c.problem == MG_MINI_RENDER)
          np = std_max(np, T(0));  // problems.cpp:228
      }
      params[j] = np;
    }
    __syncthreads();
  }
  // converged status (harness.cpp:191-198) on the last recorded params (= prev)
  double fin[3];
  block_sums3(d, [&](int j, int) {
    const double e = double(prev[j]) - k.truth[j];
    return e * e;
  }, fin, sw, c.problem != MG_MINI_RENDER);
  if (threadIdx.x == 0) {
    if (status != 2 && c.converge_threshold > 0.0 && iters_run > 0 &&
        sqrt(fin[0]) < c.converge_threshold)
      status = 1;
    mg_run_record rec;
    rec.iterations_run = iters_run;
    rec.status = status;
    rec.draws_used = draws;
    rec.evals_used = evals;
    k.recs[r] = rec;
  }
  if (k.final_params)
    for (int j = threadIdx.x; j < d; j += kThreads) k.final_params[off + j] = double(prev[j]);
}

// --------------------------------------------- one replicate per cluster
// run_single (harness.cpp:90-200) of ONE mini-render replicate spread over a
// thread-block cluster instead of one CTA, for the few-replicate case (the
// S1 configuration: P = 4096, 200 iterations, one replicate would otherwise
// use 1 of 148 SMs).  CTA rank 0 is the producer: it runs the replicate's
// exact std::mt19937_64 stream (Rng::stream, rng.hpp:23-36) and writes each
// iteration's D uniforms to global memory (L2-resident), publishing its
// progress with a release store.  Ranks 1..NC-1 are consumers: each owns a
// contiguous pixel range with the whole optimiser state in REGISTERS for
// the entire run, and per iteration computes the sample pair
// (problems.cpp:197-217), Moment2 x2, MetaEstimator::step / Adam::step,
// the record of `coord`, and the update + projection.  The four sums the
// next iteration needs (step norm and loss of the new parameters, all
// finite, params == prev) are block-reduced and exchanged through
// distributed shared memory: every consumer stores its partials into every
// consumer's slot and arrives on that CTA's mbarrier; each then sums the
// slots in rank order, so all consumers hold identical totals (fixed order:
// deterministic) after ONE exchange per iteration.
constexpr int kClusterMax = 16;
constexpr int kPPT = 4;  // pixels per consumer thread (registers)

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(out) : "r"(uint32_t(__cvta_generic_to_shared(p))), "r"(rank));
  return out;
}
__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void arrive_cluster(uint32_t bar_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_addr)
               : "memory");
}
__device__ __forceinline__ bool try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(uint32_t(__cvta_generic_to_shared(bar))), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_init_cta(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(uint32_t(__cvta_generic_to_shared(bar))),
               "r"(count) : "memory");
}

// The producer: the replicate's std::mt19937_64 state words w[312 + o]
// (o = 0 .. total-1; output o of the engine is temper(w[312 + o]), as after
// libstdc++'s seeding, random.tcc:328-343, whose first call twists) written
// RAW to `out`; the consumers temper and convert them (rng.hpp:28) as they
// read them.  The state recurrence w[j] = w[j-156] ^ mag(w[j-312],
// w[j-311]) (the twist of random.tcc:399 in sequential form) advances in
// chunks of 156 words, each depending only on the two chunks before it:
// warp 0 computes the chunks (5 words per lane, registers only, one
// __syncwarp per chunk) and stores them straight to global memory; after
// every batch of kBatchChunks chunks its lane 0 publishes the batch count in
// shared memory (release, CTA scope) and warp 1 turns that into the global
// progress word the consumers acquire (release, GPU scope, every
// kPublishBatches batches), so no fence ever stalls the twister.  The
// producer CTA's other warps idle: the twister owns its SM sub-partition's
// issue slots (warps share a scheduler by index mod 4; warps spinning there
// cost it half its rate).
constexpr int kChunkW = kMtM;                    // 156 words per chunk
#ifndef MG_S1_BATCH_CHUNKS
#define MG_S1_BATCH_CHUNKS 16
#endif
constexpr int kBatchChunks = MG_S1_BATCH_CHUNKS;  // chunks per published batch
constexpr int kBatchWords = kBatchChunks * kChunkW;
#ifndef MG_S1_PUBLISH_BATCHES
#define MG_S1_PUBLISH_BATCHES 4
#endif
constexpr int kPublishBatches = MG_S1_PUBLISH_BATCHES;
#ifndef MG_PRODUCER_PROBE
#define MG_PRODUCER_PROBE 0  // 2: the twister skips its arithmetic (probe builds)
#endif

__device__ __forceinline__ void st_release_cta_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(uint32_t(__cvta_generic_to_shared(p))),
               "r"(v)
               : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_cta_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];"
               : "=r"(v)
               : "r"(uint32_t(__cvta_generic_to_shared(p)))
               : "memory");
  return v;
}

// words the producer writes for `total` outputs: whole batches
__host__ __device__ constexpr int64_t raw_stream_words(int64_t total) {
  return (total + kBatchWords - 1) / kBatchWords * kBatchWords;
}

// seedbuf: kMtN shared words; s_done: shared batch counter.  out: at least
// raw_stream_words(total) words.
template <int CT>
__device__ void produce_raw(uint64_t* seedbuf, unsigned int* s_done, uint64_t seed, uint64_t rep,
                            int64_t total, uint64_t* out, unsigned long long* progress) {
  if (threadIdx.x == 0) {
    // Rng::stream(seed, rep) (rng.hpp:23-25): w[0..311] = chunks -2, -1
    uint64_t x = mg_mix64_dev(mg_mix64_dev(seed) ^ (rep + 0x51ed2701e35f3a6dULL));
    seedbuf[0] = x;
    for (int i = 1; i < kMtN; ++i) {
      x ^= x >> 62;
      x = 6364136223846793005ULL * x + static_cast<uint64_t>(i);
      seedbuf[i] = x;
    }
    *s_done = 0u;
  }
  __syncthreads();
  const int64_t chunks = (total + kChunkW - 1) / kChunkW;
  const int64_t batches = (chunks + kBatchChunks - 1) / kBatchChunks;
  if (threadIdx.x < 32) {  // twister warp
    // Lane l owns the contiguous words t = 5l .. 5l+4 (t < 156; lane 31
    // owns t = 155 only) of every chunk and keeps them for the last two
    // chunks in registers.  Word t of chunk k needs words t of chunks k-1
    // and k-2 and word t+1 of chunk k-2 — in-lane except for the last word
    // of a lane (lane l+1's first word, shuffled from two chunks back, off
    // the critical path) and t = 155 (word 0 of chunk k-1, one shuffle).
    const int l = threadIdx.x;
    const int t0 = 5 * l;
    const int nw_l = l < 31 ? 5 : 1;  // words owned (lane 31: t = 155)
    uint64_t v1[5], v2[5];            // chunks k-1, k-2
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      v2[q] = q < nw_l ? seedbuf[t0 + q] : 0ull;
      v1[q] = q < nw_l ? seedbuf[kChunkW + t0 + q] : 0ull;
    }
    uint64_t* wp = out + t0;  // this lane's words of the current chunk
    for (int64_t b = 0; b < batches; ++b) {
#if MG_PRODUCER_PROBE != 2
      // unrolled: the two-chunk register rotation resolves at compile time
      // (as a loop it cost ~20 moves per chunk)
#pragma unroll
      for (int kc = 0; kc < kBatchChunks; ++kc) {
        // word t0 + 5 of chunk k-2 (lane l+1's first) and word 0 of chunk k-1
        const uint64_t right = __shfl_down_sync(0xffffffffu, v2[0], 1);
        const uint64_t head1 = __shfl_sync(0xffffffffu, v1[0], 0);
        uint64_t v0[5];
#pragma unroll
        for (int q = 0; q < 4; ++q) v0[q] = v1[q] ^ mt_mag(v2[q], v2[q + 1]);
        v0[4] = v1[4] ^ mt_mag(v2[4], right);
        if (l == 31) v0[0] = v1[0] ^ mt_mag(v2[0], head1);  // t = 155
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          if (q < nw_l) wp[q] = v0[q];  // out holds whole batches (padded)
          v2[q] = v1[q];
          v1[q] = v0[q];
        }
        wp += kChunkW;
      }
#endif
      __syncwarp();  // the batch's stores precede lane 0's release
      if (l == 0) st_release_cta_u32(s_done, unsigned(b + 1));
    }
  } else if (threadIdx.x == 32) {  // publisher (warp 1, another sub-partition)
    int64_t pub = 0;
    while (pub < batches) {
      const int64_t want = pub + kPublishBatches < batches ? pub + kPublishBatches : batches;
      unsigned int done;
      while ((done = ld_acquire_cta_u32(s_done)) < unsigned(want)) {
      }
      pub = done;
      const int64_t words = pub * kBatchWords < total ? pub * kBatchWords : total;
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(progress),
                   "l"((unsigned long long)words)
                   : "memory");
    }
  }
}

// CT threads per CTA, PPT pixels per consumer thread (registers)
template <class T, int CT, int PPT>
__global__ void __launch_bounds__(CT) run_cluster_kernel(RunK<T> k, double* ubuf_all,
                                                               unsigned long long* progress_all) {
  __shared__ uint64_t seedbuf[kMtN];
  __shared__ unsigned int s_done;
  __shared__ double sw[CT / 32];
  __shared__ double xch[2][kClusterMax][4];  // [parity][source rank][sum]
  __shared__ double wsum[CT / 32][4];
  __shared__ unsigned long long s_seen;  // producer progress acquired so far
  __shared__ __align__(8) uint64_t xbar[2];
  __shared__ double tot[4];
  const mg_experiment_config& c = k.cfg;
  const uint32_t rank = cluster_rank(), NC = cluster_size(), M = NC - 1;
  MG_DCHECK(NC >= 2 && NC <= uint32_t(kClusterMax) && blockDim.x == unsigned(CT));
  const int r = blockIdx.x / NC;  // replicate within the launch
  const int d = k.dim, iters = c.iterations, spp = c.spp;
  const int64_t D = k.D;
  double* ubuf = ubuf_all + size_t(r) * raw_stream_words(int64_t(iters) * D);
  unsigned long long* progress = progress_all + r;
  if (threadIdx.x == 0) {
    s_seen = 0;
    mbar_init_cta(&xbar[0], M);
    mbar_init_cta(&xbar[1], M);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster_sync_all();  // every CTA of the cluster is running and initialised

  if (rank == 0) {  // ------------------------------------------ producer
    produce_raw<CT>(seedbuf, &s_done, c.seed, uint64_t(k.rep_begin + r), int64_t(iters) * D,
                    reinterpret_cast<uint64_t*>(ubuf), progress);
    cluster_sync_all();
    return;
  }
  // ------------------------------------------------------------ consumers
  const int me = int(rank) - 1;
  const int lo = int((int64_t(d) * me) / M), hi = int((int64_t(d) * (me + 1)) / M);
  const bool use_meta = c.optimizer == MG_OPT_META;
  const bool per_param = c.diff_norm == MG_DIFF_NORM_PER_PARAM;
  T p[PPT], pv[PPT], m2p[PPT], m2d[PPT], mean[PPT], var[PPT], ap[PPT];
  double bj[PPT], tj[PPT];
  bool own[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int j = lo + int(threadIdx.x) + q * CT;
    own[q] = j < hi;
    bj[q] = own[q] ? k.exponents[j] : 0.0;
    tj[q] = own[q] ? k.truth[j] : 0.0;
    p[q] = pv[q] = T(own[q] ? k.init[j] : 0.0);
    m2p[q] = m2d[q] = mean[q] = var[q] = ap[q] = T(0);
  }
  // cluster-wide sums of 4 per-thread values; identical in every consumer
  int xi = 0;  // exchange counter (parity = xi & 1, phase = (xi >> 1) & 1)
  auto exchange = [&](double a0, double a1, double a2, double a3) {
    // one fixed-shape block tree for the four sums (warp shuffles, then
    // warp 0 over the warp partials)
    double v[4] = {a0, a1, a2, a3};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] += __shfl_down_sync(0xffffffffu, v[q], o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 4; ++q) wsum[warp][q] = v[q];
    __syncthreads();
    const int par = xi & 1;
    if (warp == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double x = lane < CT / 32 ? wsum[lane][q] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        v[q] = __shfl_sync(0xffffffffu, x, 0);
      }
      // lane t < M stores this CTA's sums into consumer t+1's slot and
      // arrives on its barrier: the M remote round trips run in parallel
      if (lane < int(M)) {
        const uint32_t dst = uint32_t(lane) + 1;
        const uint32_t slot = map_rank(&xch[par][rank][0], dst);
#pragma unroll
        for (int q = 0; q < 4; ++q) st_cluster_f64(slot + 8u * q, v[q]);
        arrive_cluster(map_rank(&xbar[par], dst));
      }
      if (lane == 0) {
        while (!try_wait_cluster(&xbar[par], uint32_t((xi >> 1) & 1))) {
        }
        double t[4] = {0.0, 0.0, 0.0, 0.0};
        for (uint32_t src = 1; src < NC; ++src)
#pragma unroll
          for (int q = 0; q < 4; ++q) t[q] += xch[par][src][q];
#pragma unroll
        for (int q = 0; q < 4; ++q) tot[q] = t[q];
      }
    }
    ++xi;
    __syncthreads();
  };
  // sums over the initial parameters: loss, all finite
  {
    double l = 0.0, nf = 0.0;
#pragma unroll
    for (int q = 0; q < PPT; ++q)
      if (own[q]) {
        const double e = double(p[q]) - tj[q];
        l += e * e;
        nf += isfinite(double(p[q])) ? 0.0 : 1.0;
      }
    exchange(0.0, l, nf, 0.0);
  }
  double ssn = 0.0, loss = tot[1], loss_rec = 0.0;
  bool finite = tot[2] == 0.0, same_pp = true;  // params == prev at the start
  double pf_pow = 1.0, pd_pow = 1.0, b1p = 1.0, b2p = 1.0;
  int64_t pf_cnt = 0, pd_cnt = 0, t_adam = 0;
  bool meta_first = true;
  int status = 0, iters_run = 0;
  int64_t draws = 0, evals = 0;
  const int coord = c.coord;
  for (int i = 0; i < iters; ++i) {
    if (!finite) {  // harness.cpp:116-119
      status = 2;
      break;
    }
    const bool same = use_meta ? same_pp : true;
    loss_rec = loss;
    {  // this iteration's uniforms are drawn: poll only when the progress
       // seen so far (acquired, then published by a barrier) falls short —
       // the producer runs ahead, so after the first iterations never
      const unsigned long long need = (unsigned long long)(i + 1) * (unsigned long long)D;
      if (s_seen < need) {  // uniform: s_seen changes only before a barrier
        __syncthreads();
        if (threadIdx.x == 0) {
          unsigned long long v;
          do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(progress) : "memory");
          } while (v < need);
          s_seen = v;
        }
        __syncthreads();
      }
    }
    // raw engine words: temper + uniform() here (rng.hpp:28)
    const unsigned long long* u = reinterpret_cast<const unsigned long long*>(ubuf) + size_t(i) * D;
    const bool two_point = use_meta && !same_pp;  // :129
    draws += D;
    evals += D * (two_point ? 2 : 1);
    // Moment2 / Adam scalars (moment2.hpp:34-38, adam.hpp:29-31), uniform
    const bool pf_first = pf_cnt == 0;
    double cp = 0.0, cd = 0.0, norm = 0.0;
    const bool active = ssn > 0.0;
    const bool pd_had = pd_cnt > 0;
    if (use_meta) {
      pf_cnt += 1;
      pf_pow = pf_pow * c.beta_f;
      cp = (1.0 - c.beta_f) / (1.0 - pf_pow);
      if (active) {
        pd_cnt += 1;
        pd_pow = pd_pow * c.beta_delta;
      }
      cd = (1.0 - c.beta_delta) / (1.0 - pd_pow);
      norm = sqrt(ssn);
    }
    const bool adam_first = t_adam == 0;
    if (!use_meta) {
      t_adam += 1;
      b1p = b1p * c.beta1;
      b2p = b2p * c.beta2;
    }
    double a_ssn = 0.0, a_loss = 0.0, a_nf = 0.0, a_ne = 0.0;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      if (!own[q]) continue;
      const int j = lo + int(threadIdx.x) + q * CT;
      MG_DCHECK(j < hi && hi <= d);
      // sample_pair (problems.cpp:197-217)
      T cross, mb;
      const unsigned long long* uj = u + size_t(j) * spp;
      minirender_terms_fn<T>(
          bj[q], spp, [&](int s) { return mt_uniform(mt_temper(__ldcg(uj + s))); }, cross, mb);
      const T a = p[q];
      const T prop = (T(2) * a) * cross - (T(2) * T(tj[q])) * mb;
      const T diff = same ? T(0) : (T(2) * (a - (use_meta ? pv[q] : a))) * cross;
      T mest, vest, al = T(0), dl;
      if (use_meta) {
        const T m2p_old = pf_first ? T(0) : m2p[q];
        const T m2pv = m2p_old + T(cp) * (prop * prop - m2p_old);  // :144
        m2p[q] = m2pv;
        T m2dv = pd_had ? m2d[q] : T(0);
        T var_diff = T(0);
        if (per_param) {  // :146-151
          const T cs = fabs(p[q] - pv[q]);
          if (active) {
            const T tiny = sizeof(T) == 8 ? T(1e-150) : T(1e-37);
            const T xd = diff / std_max(cs, tiny);
            m2dv = m2dv + T(cd) * (xd * xd - m2dv);
            m2d[q] = m2dv;
          }
          if (pd_cnt > 0) var_diff = m2dv * (cs * cs);
        } else {  // :153-157
          if (active) {
            const T xd = diff / T(norm);
            m2dv = m2dv + T(cd) * (xd * xd - m2dv);
            m2d[q] = m2dv;
          }
          if (pd_cnt > 0) var_diff = m2dv * T(ssn);
        }
        T m = (meta_first ? T(0) : mean[q]) + diff;  // meta.hpp:92-112
        T v = (meta_first ? T(0) : var[q]) + var_diff;
        const T a_prev = meta_first ? T(-INFINITY) : ap[q];
        al = m2pv / ((m2pv + v) + T(c.eps_alpha));
        if (!c.no_alpha_clip) al = std_min(al, T(1) / (T(2) - a_prev));
        ap[q] = al;
        const T om = T(1) - al;
        m = al * m + om * prop;
        v = (al * al) * v + (om * om) * m2pv;
        mean[q] = m;
        var[q] = v;
        mest = m;
        vest = v;
        dl = (T(-c.lr) * m) / (sqrt(v) + T(c.eps_step));
      } else {  // Adam (adam.hpp:23-37); m2p/m2d hold m/v
        const T c1 = T(1.0 - c.beta1), c2 = T(1.0 - c.beta2);
        const T d1 = T(1.0 - b1p), d2 = T(1.0 - b2p);
        const T mm = T(c.beta1) * (adam_first ? T(0) : m2p[q]) + c1 * prop;
        const T vv = T(c.beta2) * (adam_first ? T(0) : m2d[q]) + c2 * (prop * prop);
        m2p[q] = mm;
        m2d[q] = vv;
        mest = mm / d1;
        vest = vv / d2;
        dl = (T(-c.lr) * mest) / (sqrt(vest) + T(c.adam_eps));
      }
      if (j == coord) {  // record iteration i (harness.cpp:170-180)
        const size_t at = size_t(r) * iters + i;
        const double x = double(a);
        const double vals[kNumSeries] = {sqrt(loss), loss, double(prop), double(diff),
                                         double(mest), double(vest),
                                         use_meta ? double(al) : nan(""), double(dl),
                                         2.0 * (x - tj[q]), ssn, x};
        for (int sx = 0; sx < kNumSeries; ++sx)
          if (k.series[sx]) k.series[sx][at] = vals[sx];
      }
      // prev = params; params += delta; project (harness.cpp:182-188, problems.cpp:228)
      const T np = std_max(a + dl, T(0));
      pv[q] = a;
      p[q] = np;
      const double dd = double(np) - double(a);
      a_ssn += dd * dd;
      const double e = double(np) - tj[q];
      a_loss += e * e;
      a_nf += isfinite(double(np)) ? 0.0 : 1.0;
      a_ne += (np == a) ? 0.0 : 1.0;
    }
    if (use_meta) meta_first = false;
    iters_run = i + 1;
    exchange(a_ssn, a_loss, a_nf, a_ne);
    same_pp = tot[3] == 0.0;
    ssn = (use_meta && !same_pp) ? tot[0] : 0.0;  // problems.cpp:206-209, 214 (Adam: no FD)
    loss = tot[1];
    finite = tot[2] == 0.0;
  }
  // final params = prev = the last recorded params (harness.cpp:116-119,
  // 182-188); converged status (harness.cpp:191-198) on their loss
  if (k.final_params)
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int j = lo + int(threadIdx.x) + q * CT;
      if (own[q]) k.final_params[size_t(r) * d + j] = double(pv[q]);
    }
  if (me == 0 && threadIdx.x == 0) {
    if (status != 2 && c.converge_threshold > 0.0 && iters_run > 0 &&
        sqrt(loss_rec) < c.converge_threshold)
      status = 1;
    mg_run_record rec;
    rec.iterations_run = iters_run;
    rec.status = status;
    rec.draws_used = draws;
    rec.evals_used = evals;
    k.recs[r] = rec;
  }
  cluster_sync_all();
}

// The producer alone (probe for tools/s1_producer_probe.py): one CTA of CT
// threads streams `total` uniforms of Rng::stream(seed, rep) into out.
template <int CT>
__global__ void __launch_bounds__(CT) mt_stream_probe_kernel(uint64_t seed, uint64_t rep,
                                                             int64_t total, double* out,
                                                             unsigned long long* progress) {
  __shared__ uint64_t seedbuf[kMtN];
  __shared__ unsigned int s_done;
  produce_raw<CT>(seedbuf, &s_done, seed, rep, total, reinterpret_cast<uint64_t*>(out), progress);
}

// Shape of the one-replicate-per-cluster runner: cluster size (16 CTAs, 15
// consumers, when the device can co-schedule them, else 8) and CTA shape
// (512 threads x 2 pixels when the pixels fit: one pixel per thread at S1,
// else 256 x 4); nc = 0: use the one-CTA-per-replicate kernel (many
// replicates fill the GPU better that way, or the pixels do not fit the
// consumers' registers).
struct ClusterShape {
  int nc = 0, threads = 0;
};

template <class T, int CT, int PPT>
int cluster_query(mg_ctx* ctx, int nc, int R) {
  auto kernel = run_cluster_kernel<T, CT, PPT>;
  if (nc > 8 &&
      cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(unsigned(R * nc));
  lc.blockDim = dim3(CT);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(nc);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, kernel, &lc) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return clusters;
}

template <class T>
ClusterShape cluster_shape_query(mg_ctx* ctx, int d, int R) {
#ifndef MG_S1_NC_FIRST
#define MG_S1_NC_FIRST 16
#endif
  for (int nc : {MG_S1_NC_FIRST, 16, 8}) {
    if (int64_t(R) * nc > int64_t(ctx->sm_count)) continue;
    if (d <= (nc - 1) * 512 * 2 && cluster_query<T, 512, 2>(ctx, nc, R) >= R) return {nc, 512};
    if (d <= (nc - 1) * 256 * 4 && cluster_query<T, 256, 4>(ctx, nc, R) >= R) return {nc, 256};
  }
  return {};
}

// memoised per (device, d, R): the occupancy queries cost more than an S1
// run's iterations
template <class T>
ClusterShape cluster_shape(mg_ctx* ctx, int d, int R) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, ClusterShape> memo;
  const auto key = std::make_tuple(ctx->device, d, R);
  {
    std::lock_guard<std::mutex> lk(mu);
    const auto it = memo.find(key);
    if (it != memo.end()) return it->second;
  }
  const ClusterShape cs = cluster_shape_query<T>(ctx, d, R);
  std::lock_guard<std::mutex> lk(mu);
  memo[key] = cs;
  return cs;
}

// ------------------------------------------------------------- host side
int problem_dim(const mg_experiment_config* c) {
  return c->problem == MG_EXP_RATE ? 1 : (c->problem == MG_MULT_NOISE ? c->dim : c->pixel_count);
}

// TrajectorySchedule::at (problems.hpp:207-215) on the host with the
// reference's own libm exp, so scripted runs match bit for bit.
void schedule_table(const mg_experiment_config* c, const std::vector<double>& from,
                    const std::vector<double>& to, std::vector<double>& out) {
  const int d = int(from.size());
  const int horizon = c->iterations;
  out.assign(size_t(c->iterations + 1) * d, 0.0);
  for (int i = 0; i <= c->iterations; ++i) {
    int clamped = i < horizon - 1 ? i : horizon - 1;
    if (clamped < 0) clamped = 0;
    for (int j = 0; j < d; ++j) {
      double v;
      if (c->trajectory == MG_TRAJ_SCRIPTED_LINEAR) {
        const double f = horizon <= 1 ? 1.0 : double(clamped) / double(horizon - 1);
        v = from[j] + (to[j] - from[j]) * f;
      } else {
        const double e = exp(-c->traj_rate * double(clamped));
        v = to[j] + (from[j] - to[j]) * e;
      }
      out[size_t(i) * d + j] = v;
    }
  }
}

template <class T>
// stats/active non-null: every series is kept on the device and reduced
// there (aggregate.cu); only the [kNumSeries][5][iterations] statistics and
// active counts come back (`series` is ignored).
int run_replicates(mg_ctx* ctx, const mg_experiment_config* cfg, int rep_begin, int R,
                   mg_run_record* records, const mg_run_series* series, double* final_params,
                   double* stats = nullptr, int32_t* active = nullptr, double* full = nullptr) {
  MG_NVTX("run_replicates");
  const int d = problem_dim(cfg);
  const int iters = cfg->iterations;
  std::vector<double> truth(d, 0.0), init(d, 0.0);
  int64_t D = 0;
  double* dexp = nullptr;
  double* dtruth_dev = nullptr;  // mini-render: the generated target, already on the device
  cudaStream_t s = ctx->stream;
  std::vector<void*> allocs;
  auto dalloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return p;
  };
  auto cleanup = [&]() {
    for (void* p : allocs) cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
  };
  switch (cfg->problem) {
    case MG_EXP_RATE:  // problems.cpp:30-42
      if (!(cfg->target_mean > 0.0)) return fail(MG_EINVAL, "exp-rate: target mean must be positive");
      if (cfg->samples_per_iter < 2)
        return fail(MG_EINVAL, "exp-rate: samples_per_iter must be at least 2");
      if (!(cfg->rate_init > 0.0)) return fail(MG_EINVAL, "exp-rate: initial rate must be positive");
      truth[0] = 1.0 / cfg->target_mean;
      init[0] = cfg->rate_init;
      D = cfg->samples_per_iter;
      break;
    case MG_MULT_NOISE:  // problems.cpp:99-108 with target 0 (harness.cpp:71-73)
      if (d < 1) return fail(MG_EINVAL, "mult-noise: empty target");
      if (cfg->sigma < 0.0) return fail(MG_EINVAL, "mult-noise: noise amplitude must be >= 0");
      if (cfg->samples_per_iter < 1)
        return fail(MG_EINVAL, "mult-noise: samples_per_iter must be >= 1");
      for (int j = 0; j < d; ++j) init[j] = truth[j] + 2.0;
      D = int64_t(cfg->samples_per_iter) * d;
      break;
    default: {  // mini-render problems.cpp:162-175
      if (d < 1) return fail(MG_EINVAL, "mini-render: pixel_count must be >= 1");
      if (cfg->spp < 2) return fail(MG_EINVAL, "mini-render: spp must be at least 2");
      dexp = (double*)dalloc(sizeof(double) * d);
      double* dT = (double*)dalloc(sizeof(double) * d);
      if (!dexp || !dT) {
        cleanup();
        return fail(MG_ENOMEM, "run: allocation failed");
      }
      int st = mg_minirender_generate(ctx, d, cfg->problem_seed, cfg->exponent_max, dexp, dT);
      if (st) {
        cleanup();
        return st;
      }
      // the device copy serves as the run's truth; the host needs it only
      // for a scripted trajectory's schedule (no synchronous round trip)
      if (cfg->trajectory != MG_TRAJ_OPTIMISE)
        MG_CUDA_TRY(cudaMemcpy(truth.data(), dT, sizeof(double) * d, cudaMemcpyDeviceToHost));
      else
        dtruth_dev = dT;
      for (int j = 0; j < d; ++j) init[j] = cfg->albedo_init;
      D = int64_t(d) * cfg->spp;
    }
  }
  if (cfg->coord >= d) {
    cleanup();
    return fail(MG_EINVAL, "coord exceeds problem dimension");
  }
  RunK<T> k{};
  k.cfg = *cfg;
  k.dim = d;
  k.D = D;
  k.rep_begin = rep_begin;
  k.R = R;
  k.exponents = dexp;
  double* dtruth = dtruth_dev ? dtruth_dev : (double*)dalloc(sizeof(double) * d);
  double* dinit = (double*)dalloc(sizeof(double) * d);
  if (!dtruth || !dinit) {
    cleanup();
    return fail(MG_ENOMEM, "run: allocation failed");
  }
  if (!dtruth_dev)
    cudaMemcpyAsync(dtruth, truth.data(), sizeof(double) * d, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(dinit, init.data(), sizeof(double) * d, cudaMemcpyHostToDevice, s);
  k.truth = dtruth;
  k.init = dinit;
  std::vector<double> sched;
  if (cfg->trajectory != MG_TRAJ_OPTIMISE) {
    schedule_table(cfg, init, truth, sched);
    double* dsched = (double*)dalloc(sizeof(double) * sched.size());
    if (!dsched) {
      cleanup();
      return fail(MG_ENOMEM, "run: allocation failed");
    }
    cudaMemcpyAsync(dsched, sched.data(), sizeof(double) * sched.size(), cudaMemcpyHostToDevice, s);
    k.sched = dsched;
  }
  const size_t vec_bytes = sizeof(T) * size_t(R) * d;
  T** vecs[] = {&k.params, &k.prev, &k.prop, &k.diff, &k.iprop, &k.idiff, &k.m2p, &k.m2d,
                &k.mean, &k.var, &k.ap, &k.am, &k.av, &k.delta, &k.mest, &k.vest};
  for (T** v : vecs) {
    *v = (T*)dalloc(vec_bytes);
    if (!*v) {
      cleanup();
      return fail(MG_ENOMEM, "run: allocation failed");
    }
  }
  k.ubuf = (double*)dalloc(sizeof(double) * size_t(R) * D);
  k.recs = (mg_run_record*)dalloc(sizeof(mg_run_record) * R);
  if (!k.ubuf || !k.recs) {
    cleanup();
    return fail(MG_ENOMEM, "run: allocation failed");
  }
  const size_t ser_bytes = sizeof(double) * size_t(R) * iters;
  void* const* host_series = series && !stats ? reinterpret_cast<void* const*>(series) : nullptr;
  double* dstats = nullptr;
  int32_t* dactive = nullptr;
  if (stats) {
    double* base = (double*)dalloc(ser_bytes * kNumSeries);
    dstats = (double*)dalloc(sizeof(double) * 5 * kNumSeries * size_t(iters));
    dactive = (int32_t*)dalloc(sizeof(int32_t) * size_t(iters));
    if (!base || !dstats || !dactive) {
      cleanup();
      return fail(MG_ENOMEM, "run: allocation failed");
    }
    cudaMemsetAsync(base, 0xff, ser_bytes * kNumSeries, s);
    for (int i = 0; i < kNumSeries; ++i) k.series[i] = base + size_t(i) * R * iters;
  }
  for (int i = 0; i < kNumSeries && !stats; ++i) {
    k.series[i] = nullptr;
    if (host_series && host_series[i]) {
      k.series[i] = (double*)dalloc(ser_bytes);
      if (!k.series[i]) {
        cleanup();
        return fail(MG_ENOMEM, "run: allocation failed");
      }
      // entries past iterations_run stay NaN (0xff.. bytes = NaN)
      cudaMemsetAsync(k.series[i], 0xff, ser_bytes, s);
    }
  }
  if (final_params) {
    k.final_params = (double*)dalloc(sizeof(double) * size_t(R) * d);
    if (!k.final_params) {
      cleanup();
      return fail(MG_ENOMEM, "run: allocation failed");
    }
  }
  const size_t full_bytes = sizeof(double) * size_t(R) * iters * 8 * size_t(d);
  if (full) {
    k.full = (double*)dalloc(full_bytes);
    if (!k.full) {
      cleanup();
      return fail(MG_ENOMEM, "run: allocation failed (full records)");
    }
    cudaMemsetAsync(k.full, 0xff, full_bytes, s);  // NaN past iterations_run
  }
  // few replicates of a mini-render run: one cluster per replicate
  ClusterShape cs;
  if (g_cluster_runner && cfg->problem == MG_MINI_RENDER && cfg->trajectory == MG_TRAJ_OPTIMISE &&
      !cfg->independent_variance_samples && !full &&
      sizeof(double) * size_t(R) * iters * D <= (size_t(1) << 30))
    cs = cluster_shape<T>(ctx, d, R);
  if (cs.nc > 0) {
    double* ubuf = (double*)dalloc(sizeof(double) * size_t(R) * raw_stream_words(int64_t(iters) * D));
    auto* progress = (unsigned long long*)dalloc(sizeof(unsigned long long) * size_t(R));
    if (!ubuf || !progress) {
      cleanup();
      return fail(MG_ENOMEM, "run: allocation failed (cluster runner)");
    }
    cudaMemsetAsync(progress, 0, sizeof(unsigned long long) * size_t(R), s);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(unsigned(R * cs.nc));
    lc.blockDim = dim3(unsigned(cs.threads));
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(cs.nc);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaError_t le = cs.threads == 512
                         ? cudaLaunchKernelEx(&lc, run_cluster_kernel<T, 512, 2>, k, ubuf, progress)
                         : cudaLaunchKernelEx(&lc, run_cluster_kernel<T, 256, 4>, k, ubuf, progress);
    if (le != cudaSuccess) {
      cleanup();
      return cuda_fail(le, "run_cluster_kernel");
    }
  } else {
    run_kernel<T><<<R, kThreads, 0, s>>>(k);
  }
  ctx->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "run_kernel");
  }
  if (stats) {
    static_assert(sizeof(mg_run_record) % sizeof(int32_t) == 0, "record stride");
    const int st = launch_aggregate(ctx, kNumSeries, R, iters, k.series[0],
                                    &k.recs[0].iterations_run,
                                    int(sizeof(mg_run_record) / sizeof(int32_t)), dstats, dactive);
    if (st) {
      cleanup();
      return st;
    }
    cudaMemcpyAsync(stats, dstats, sizeof(double) * 5 * kNumSeries * size_t(iters),
                    cudaMemcpyDeviceToHost, s);
    if (active)
      cudaMemcpyAsync(active, dactive, sizeof(int32_t) * size_t(iters), cudaMemcpyDeviceToHost, s);
  }
  cudaMemcpyAsync(records, k.recs, sizeof(mg_run_record) * R, cudaMemcpyDeviceToHost, s);
  for (int i = 0; i < kNumSeries && host_series; ++i)
    if (k.series[i]) cudaMemcpyAsync(host_series[i], k.series[i], ser_bytes, cudaMemcpyDeviceToHost, s);
  if (full) cudaMemcpyAsync(full, k.full, full_bytes, cudaMemcpyDeviceToHost, s);
  if (final_params)
    cudaMemcpyAsync(final_params, k.final_params, sizeof(double) * size_t(R) * d,
                    cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  cleanup();
  if (e != cudaSuccess) return cuda_fail(e, "run_kernel execution");
  return MG_OK;
}

}  // namespace
}  // namespace mg

using namespace mg;

extern "C" int mg_mt_stream_probe(mg_ctx* ctx, uint64_t seed, uint64_t rep, int64_t total,
                                  double* out, unsigned long long* progress) {
  if (!ctx || !out || !progress || total < 1) return fail(MG_EINVAL, "mg_mt_stream_probe: bad arguments");
  // the producer writes whole batches: stream into scratch, copy `total`
  double* scratch = static_cast<double*>(ctx_scratch(ctx, sizeof(double) * raw_stream_words(total)));
  if (!scratch) return fail(MG_ENOMEM, "mg_mt_stream_probe: scratch allocation failed");
  mt_stream_probe_kernel<512><<<1, 512, 0, ctx->stream>>>(seed, rep, total, scratch, progress);
  MG_LAUNCH_CHECK(ctx);
  MG_CUDA_TRY(cudaMemcpyAsync(out, scratch, sizeof(double) * total, cudaMemcpyDeviceToDevice,
                              ctx->stream));
  return MG_OK;
}

extern "C" int mg_run_replicates_full(mg_ctx* ctx, const mg_experiment_config* cfg,
                                      int32_t rep_begin, int32_t rep_count,
                                      mg_run_record* records, const mg_run_series* series,
                                      double* final_params, double* full) {
  if (!ctx || !cfg || !records || !full)
    return fail(MG_EINVAL, "mg_run_replicates_full: null argument");
  int st = mg_config_validate(cfg);
  if (st) return st;
  if (rep_count < 1 || rep_begin < 0)
    return fail(MG_EINVAL, "mg_run_replicates_full: bad replicate range");
  if (cfg->rng != MG_RNG_MT64)
    return fail(MG_EUNSUPPORTED, "mg_run_replicates_full: only the bit-exact mt64 streams are supported");
  if (cfg->dtype == MG_F64)
    return run_replicates<double>(ctx, cfg, rep_begin, rep_count, records, series, final_params,
                                  nullptr, nullptr, full);
  return run_replicates<float>(ctx, cfg, rep_begin, rep_count, records, series, final_params,
                               nullptr, nullptr, full);
}

extern "C" int mg_run_experiment_stats(mg_ctx* ctx, const mg_experiment_config* cfg,
                                       int32_t rep_begin, int32_t rep_count,
                                       mg_run_record* records, double* stats, int32_t* active) {
  if (!ctx || !cfg || !records || !stats)
    return fail(MG_EINVAL, "mg_run_experiment_stats: null argument");
  int st = mg_config_validate(cfg);
  if (st) return st;
  if (rep_count < 1 || rep_begin < 0)
    return fail(MG_EINVAL, "mg_run_experiment_stats: bad replicate range");
  if (cfg->rng != MG_RNG_MT64)
    return fail(MG_EUNSUPPORTED, "mg_run_experiment_stats: only the bit-exact mt64 streams are supported");
  if (cfg->dtype == MG_F64)
    return run_replicates<double>(ctx, cfg, rep_begin, rep_count, records, nullptr, nullptr, stats,
                                  active);
  return run_replicates<float>(ctx, cfg, rep_begin, rep_count, records, nullptr, nullptr, stats,
                               active);
}

extern "C" int mg_run_replicates(mg_ctx* ctx, const mg_experiment_config* cfg, int32_t rep_begin,
                                 int32_t rep_count, mg_run_record* records,
                                 const mg_run_series* series, double* final_params) {
  if (!ctx || !cfg || !records) return fail(MG_EINVAL, "mg_run_replicates: null argument");
  int st = mg_config_validate(cfg);
  if (st) return st;
  if (rep_count < 1 || rep_begin < 0) return fail(MG_EINVAL, "mg_run_replicates: bad replicate range");
  if (cfg->rng != MG_RNG_MT64)
    return fail(MG_EUNSUPPORTED, "mg_run_replicates: only the bit-exact mt64 streams are supported");
  if (cfg->dtype == MG_F64)
    return run_replicates<double>(ctx, cfg, rep_begin, rep_count, records, series, final_params);
  return run_replicates<float>(ctx, cfg, rep_begin, rep_count, records, series, final_params);
}
