/*
 * metagrad_oracle.c — CPU restatement (plain C, fp64, sequential) of the
 * reference metagrad hot path.  TEST INFRASTRUCTURE ONLY: the checker for the
 * CUDA path (see metagrad_oracle.h).  Pinned against tests/golden/, which
 * oracle/gen_golden.py generates from the unmodified reference (oracle/_ref).
 *
 * The F1 path-tracing sections (mgo_quad_*, mgo_helix_*, mgo_mesh*_*) have
 * NO reference counterpart (the reference has no renderer):
 * parity unpinned against the reference; they restate this repo's own
 * specification and are checked by finite differences,
 * unbiasedness tests and brute-force intersection instead.
 *
 * Build: make -C oracle  (gcc -O2 -ffp-contract=off; no -march: the
 * reference's Release build performs no FMA contraction).
 */
#include "metagrad_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ RNG */

/* rng.hpp:9-14 */
uint64_t mgo_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* std::mt19937_64 = mersenne_twister_engine<uint64_t, 64, 312, 156, 31,
 * 0xb5026f5aa96619e9, 29, 0x5555555555555555, 17, 0x71d67fffeda60000, 37,
 * 0xfff7eee000000000, 43, 6364136223846793005> (libstdc++ random.h:1620-1627).
 * seed(): random.tcc:328-343; _M_gen_rand (twist): random.tcc:399;
 * operator(): random.tcc:455-470. */
enum { MT_N = 312, MT_M = 156 };
#define MT_A 0xb5026f5aa96619e9ULL
#define MT_UPPER 0xffffffff80000000ULL
#define MT_LOWER 0x000000007fffffffULL

void mgo_mt64_seed(mgo_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    uint64_t x = g->mt[i - 1];
    x ^= x >> 62;
    g->mt[i] = 6364136223846793005ULL * x + (uint64_t)i;
  }
  g->idx = MT_N;
}

static void mt_twist(mgo_mt64* g) {
  uint64_t* mt = g->mt;
  for (int k = 0; k < MT_N; ++k) {
    const uint64_t y = (mt[k] & MT_UPPER) | (mt[(k + 1) % MT_N] & MT_LOWER);
    mt[k] = mt[(k + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
  }
  g->idx = 0;
}

uint64_t mgo_mt64_next(mgo_mt64* g) {
  if (g->idx >= MT_N) mt_twist(g);
  uint64_t z = g->mt[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71d67fffeda60000ULL;
  z ^= (z << 37) & 0xfff7eee000000000ULL;
  z ^= z >> 43;
  return z;
}

/* rng.hpp:23-25 */
void mgo_rng_stream(mgo_mt64* g, uint64_t base_seed, uint64_t replicate) {
  mgo_mt64_seed(g, mgo_mix64(mgo_mix64(base_seed) ^ (replicate + 0x51ed2701e35f3a6dULL)));
}

/* rng.hpp:28 */
double mgo_uniform(mgo_mt64* g) { return (double)(mgo_mt64_next(g) >> 11) * 0x1.0p-53; }
/* rng.hpp:31 */
double mgo_uniform_pos(mgo_mt64* g) { return 1.0 - mgo_uniform(g); }

void mgo_rng_draws(uint64_t seed, uint64_t rep, int mode, int64_t n, void* out) {
  mgo_mt64 g;
  if (mode == 0 || mode == 4)
    mgo_mt64_seed(&g, seed);
  else
    mgo_rng_stream(&g, seed, rep);
  uint64_t* u = (uint64_t*)out;
  double* d = (double*)out;
  for (int64_t i = 0; i < n; ++i) {
    if (mode == 0 || mode == 1)
      u[i] = mgo_mt64_next(&g);
    else if (mode == 2 || mode == 4)
      d[i] = mgo_uniform(&g);
    else
      d[i] = mgo_uniform_pos(&g);
  }
}

/* GF(2) jump-ahead (Haramoto et al. 2008) restated bit by bit: for a
 * generator at a block boundary (idx == 312, window W = mt[0..311]),
 * R = g(A) W with Horner's rule, A = one output step of the window
 * (x_new = W[156] ^ mag(W[0], W[1]), shift).  poly: 312 words, bit i = g_i. */
void mgo_mt64_jump(mgo_mt64* g, const uint64_t* poly, int deg) {
  uint64_t W[MT_N], R[MT_N];
  memcpy(W, g->mt, sizeof(W));
  memset(R, 0, sizeof(R));
  int s = 0;
  for (int i = deg; i >= 0; --i) {
    const uint64_t y = (R[s] & MT_UPPER) | (R[(s + 1) % MT_N] & MT_LOWER);
    R[s] = R[(s + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
    s = (s + 1) % MT_N;
    if ((poly[i >> 6] >> (i & 63)) & 1ULL)
      for (int c = 0; c < MT_N; ++c) R[(s + c) % MT_N] ^= W[c];
  }
  for (int c = 0; c < MT_N; ++c) g->mt[c] = R[(s + c) % MT_N];
  g->idx = MT_N;
}

/* Philox4x32-10 (Salmon et al., SC'11), published algorithm; the scale-mode
 * RNG of the device samplers (paper_2309_15676_b200/csrc/philox.cuh).
 * ctr/out are 4 words; key is the 64-bit replicate engine seed. */
void mgo_philox4x32_10(const uint32_t ctr[4], uint64_t key, uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* uniform s of pixel j at iteration it, stream st (philox_uniform_at) */
double mgo_philox_uniform(uint64_t key, uint32_t j, uint32_t it, uint32_t s, uint32_t st) {
  const uint32_t ctr[4] = {j, it, s >> 1, st};
  uint32_t o[4];
  mgo_philox4x32_10(ctr, key, o);
  const uint64_t a = ((uint64_t)o[0] << 21) ^ (uint64_t)(o[1] >> 11);
  const uint64_t b = ((uint64_t)o[2] << 21) ^ (uint64_t)(o[3] >> 11);
  return (double)((s & 1u) ? b : a) * 0x1.0p-53;
}

/* -------------------------------------------------------------- Moment2 */

/* moment2.hpp:30-39: count++; decay_pow *= decay; m2 += (w/w_sum)*(x^2 - m2) */
void mgo_moment2_step(int64_t n, double decay, double* decay_pow, int64_t* count, double* m2,
                      const double* x) {
  if (*count == 0) memset(m2, 0, (size_t)n * sizeof(double)); /* lazy Vec::Zero, :31 */
  ++*count;
  *decay_pow *= decay;
  const double w = 1.0 - decay;
  const double w_sum = 1.0 - *decay_pow;
  const double c = w / w_sum;
  for (int64_t i = 0; i < n; ++i) m2[i] = m2[i] + c * (x[i] * x[i] - m2[i]);
}

/* ---------------------------------------------------------- MetaEstimator */

/* min(raw, 1/(2 - alpha_prev)) with std::min semantics (meta.hpp:30-32) */
static inline double clip_alpha(double raw, double alpha_prev) {
  const double bound = 1.0 / (2.0 - alpha_prev);
  return (bound < raw) ? bound : raw;
}

/* meta.hpp:90-113 */
int mgo_meta_step(int64_t n, double lr, double eps_step, double eps_alpha, int clip, int first_call,
                  double* mean, double* var, double* alpha_prev, const double* prop,
                  const double* diff, const double* var_prop, const double* var_diff,
                  double* delta) {
  if (first_call) {
    for (int64_t i = 0; i < n; ++i) {
      mean[i] = 0.0;
      var[i] = 0.0;
      alpha_prev[i] = -INFINITY;
    }
  }
  for (int64_t i = 0; i < n; ++i)
    if (var_prop[i] < 0.0 || var_diff[i] < 0.0) return MG_ELOGIC; /* :100-101 */
  for (int64_t i = 0; i < n; ++i) {
    double m = mean[i] + diff[i];  /* :103 */
    double v = var[i] + var_diff[i]; /* :104 */
    double a = var_prop[i] / ((var_prop[i] + v) + eps_alpha); /* :106 */
    if (clip) a = clip_alpha(a, alpha_prev[i]);              /* :107 */
    alpha_prev[i] = a;                                        /* :108 */
    const double one_m = 1.0 - a;
    m = a * m + one_m * prop[i];                     /* :110 */
    v = (a * a) * v + (one_m * one_m) * var_prop[i]; /* :111 */
    mean[i] = m;
    var[i] = v;
    delta[i] = ((-lr) * m) / (sqrt(v) + eps_step); /* :112 */
  }
  return 0;
}

/* ------------------------------------------------------------------- Adam */

/* adam.hpp:23-37 */
void mgo_adam_step(int64_t n, mg_adam_scalars* s, double* m, double* v, const double* grad,
                   double* delta) {
  if (s->t == 0) {
    memset(m, 0, (size_t)n * sizeof(double));
    memset(v, 0, (size_t)n * sizeof(double));
  }
  ++s->t;
  s->beta1_pow *= s->beta1;
  s->beta2_pow *= s->beta2;
  const double c1 = 1.0 - s->beta1, c2 = 1.0 - s->beta2;
  const double d1 = 1.0 - s->beta1_pow, d2 = 1.0 - s->beta2_pow;
  for (int64_t i = 0; i < n; ++i) {
    const double g = grad[i];
    m[i] = s->beta1 * m[i] + c1 * g;
    v[i] = s->beta2 * v[i] + c2 * (g * g);
    const double mh = m[i] / d1, vh = v[i] / d2;
    if (delta) delta[i] = ((-s->lr) * mh) / (sqrt(vh) + s->eps);
  }
}

/* ---------------------------------------------- fused update iterations */

/* The reduction epilogue shared by both fused updates (sequential order). */
static void reduce_epilogue(int64_t n, const double* p_old, const double* p_new,
                            const double* target, mg_update_scalars* sc) {
  double ssn = 0.0, changed = 0.0, loss = 0.0, nonfinite = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = p_new[i] - p_old[i];
    ssn += d * d;                                    /* problems.cpp:214 */
    changed += (p_new[i] != p_old[i]) ? 1.0 : 0.0;   /* problems.cpp:206 */
    if (target) {
      const double e = p_new[i] - target[i];
      loss += e * e;                                 /* problems.cpp:225 */
    }
    nonfinite += isfinite(p_new[i]) ? 0.0 : 1.0;     /* harness.cpp:116 */
  }
  sc->ssn = ssn;
  sc->changed = changed;
  sc->loss = target ? loss : NAN;
  sc->nonfinite = nonfinite;
}

/* harness.cpp:144 (Moment2 prop), :145-158 (diff decoupling), :160
 * (MetaEstimator::step), :182-188 (update + projection). */
int mgo_meta_update(int64_t n, const mg_meta_update_args* a, const double* prop, const double* diff,
                    const double* vprop, const double* vdiff, double* m2_prop, double* m2_diff,
                    double* mean, double* var, double* alpha_prev, const double* params_in,
                    double* params_out, const double* params_prev, const double* target,
                    mg_update_scalars* sc, double* delta_out) {
  const double ssn = a->ssn_from_host ? a->ssn_host : sc->ssn;
  const double* vp = vprop ? vprop : prop;
  const double* vd = vdiff ? vdiff : diff;
  const int per_param = a->diff_norm == MG_DIFF_NORM_PER_PARAM;
  if (per_param && !params_prev) return MG_EINVAL;
  /* diff EMA scalars (moment2.hpp:34-38), stepped only when ssn > 0 */
  const int diff_active = ssn > 0.0;
  const int64_t count_before = sc->diff_count;
  double dpow = sc->diff_decay_pow;
  int64_t dcount = sc->diff_count;
  if (diff_active) {
    ++dcount;
    dpow *= a->beta_delta;
  }
  const double c_diff = (1.0 - a->beta_delta) / (1.0 - dpow);
  const double norm = sqrt(ssn); /* harness.cpp:154: diff / std::sqrt(ssn) */
  const double c_prop = a->prop_coef;
  double* p_old = (double*)malloc((size_t)n * sizeof(double));
  if (!p_old) return MG_ENOMEM;
  memcpy(p_old, params_in, (size_t)n * sizeof(double));
  for (int64_t i = 0; i < n; ++i) {
    /* Moment2(beta_f).step(prop) (moment2.hpp:38) */
    const double m2p_old = a->first_step ? 0.0 : m2_prop[i];
    const double m2p = m2p_old + c_prop * (vp[i] * vp[i] - m2p_old);
    m2_prop[i] = m2p;
    /* decoupled diff variance (harness.cpp:146-157) */
    double m2d = count_before > 0 ? m2_diff[i] : 0.0;
    double var_diff = 0.0;
    if (per_param) {
      const double cs = fabs(params_in[i] - params_prev[i]);
      if (diff_active) {
        const double x = vd[i] / ((cs < 1e-150) ? 1e-150 : cs);
        m2d = m2d + c_diff * (x * x - m2d);
        m2_diff[i] = m2d;
      }
      if (dcount > 0) var_diff = m2d * (cs * cs);
    } else {
      if (diff_active) {
        const double x = vd[i] / norm;
        m2d = m2d + c_diff * (x * x - m2d);
        m2_diff[i] = m2d;
      }
      if (dcount > 0) var_diff = m2d * ssn; /* rescale_diff_variance, meta.hpp:51-53 */
    }
    /* MetaEstimator::step (meta.hpp:103-112) */
    double m = (a->first_step ? 0.0 : mean[i]) + diff[i];
    double v = (a->first_step ? 0.0 : var[i]) + var_diff;
    const double ap = a->first_step ? -INFINITY : alpha_prev[i];
    double al = m2p / ((m2p + v) + a->meta.eps_alpha);
    if (a->meta.clip_enabled) al = clip_alpha(al, ap);
    alpha_prev[i] = al;
    const double om = 1.0 - al;
    m = al * m + om * prop[i];
    v = (al * al) * v + (om * om) * m2p;
    mean[i] = m;
    var[i] = v;
    const double delta = ((-a->meta.lr) * m) / (sqrt(v) + a->meta.eps_step);
    if (delta_out) delta_out[i] = delta;
    double p = params_in[i] + delta;
    if (a->project) p = (p < a->proj_lo) ? a->proj_lo : p; /* std::max(p, lo) */
    if (a->project == 2) p = (a->proj_hi < p) ? a->proj_hi : p;
    params_out[i] = p;
  }
  sc->ssn_used = ssn;
  sc->diff_count = dcount;
  sc->diff_decay_pow = dpow;
  reduce_epilogue(n, p_old, params_out, target, sc);
  free(p_old);
  return 0;
}

void mgo_adam_update(int64_t n, mg_adam_scalars* s, int project, double proj_lo, const double* grad,
                     double* m, double* v, const double* params_in, double* params_out,
                     const double* target, mg_update_scalars* sc) {
  double* delta = (double*)malloc((size_t)n * sizeof(double));
  double* p_old = (double*)malloc((size_t)n * sizeof(double));
  memcpy(p_old, params_in, (size_t)n * sizeof(double));
  const double ssn = sc->ssn;
  mgo_adam_step(n, s, m, v, grad, delta);
  for (int64_t i = 0; i < n; ++i) {
    double p = params_in[i] + delta[i];
    if (project) p = (p < proj_lo) ? proj_lo : p;
    params_out[i] = p;
  }
  sc->ssn_used = ssn;
  reduce_epilogue(n, p_old, params_out, target, sc);
  free(delta);
  free(p_old);
}

/* ------------------------------------------------------------ problems */

/* problems.cpp:162-173: gen = Rng(mix64(gen_seed)); all b_j, then all T_j */
void mgo_minirender_generate(int32_t pixel_count, uint64_t gen_seed, double exponent_max,
                             double* exponents, double* target) {
  mgo_mt64 g;
  mgo_mt64_seed(&g, mgo_mix64(gen_seed));
  for (int32_t j = 0; j < pixel_count; ++j) exponents[j] = exponent_max * mgo_uniform(&g);
  for (int32_t j = 0; j < pixel_count; ++j) target[j] = 0.2 + 0.8 * mgo_uniform(&g);
}

/* problems.cpp:177-195 */
void mgo_minirender_kernel_terms(int32_t pixel_count, int32_t spp, const double* exponents,
                                 const double* uniforms, double* cross, double* mean_basis) {
  const double n = (double)spp;
  for (int32_t j = 0; j < pixel_count; ++j) {
    const double b = exponents[j];
    double sum = 0.0, sum_sq = 0.0;
    for (int32_t s = 0; s < spp; ++s) {
      const double basis = (b + 1.0) * pow(uniforms[(size_t)j * spp + s], b);
      sum += basis;
      sum_sq += basis * basis;
    }
    cross[j] = (sum * sum - sum_sq) / (n * (n - 1.0));
    mean_basis[j] = sum / n;
  }
}

/* problems.cpp:197-217 */
double mgo_minirender_sample_pair(int32_t pixel_count, int32_t spp, const double* exponents,
                                  const double* target, mgo_mt64* g, const double* now,
                                  const double* prev, double* prop, double* diff) {
  const size_t draws = (size_t)pixel_count * (size_t)spp;
  double* u = (double*)malloc(draws * sizeof(double));
  double* cross = (double*)malloc((size_t)pixel_count * sizeof(double));
  double* mb = (double*)malloc((size_t)pixel_count * sizeof(double));
  for (size_t k = 0; k < draws; ++k) u[k] = mgo_uniform(g);
  mgo_minirender_kernel_terms(pixel_count, spp, exponents, u, cross, mb);
  int same = 1;
  for (int32_t j = 0; j < pixel_count; ++j) same &= (now[j] == prev[j]);
  double ssn = 0.0;
  for (int32_t j = 0; j < pixel_count; ++j) {
    prop[j] = (2.0 * now[j]) * cross[j] - (2.0 * target[j]) * mb[j]; /* :205 */
    if (same) {
      diff[j] = 0.0;
    } else {
      const double d = now[j] - prev[j];
      diff[j] = (2.0 * d) * cross[j]; /* :213 */
      ssn += d * d;                   /* :214 */
    }
  }
  free(u);
  free(cross);
  free(mb);
  return same ? 0.0 : ssn;
}

/* problems.cpp:44-52 */
double mgo_exprate_gradient_from_batch(double target_mean, int32_t samples, double rate,
                                       double sum_c, double sum_c_sq) {
  const double n = (double)samples;
  const double rate_sq = rate * rate;
  return ((-2.0) * (sum_c * sum_c - sum_c_sq)) / (((n * (n - 1.0)) * rate_sq) * rate) +
         ((2.0 * target_mean) * sum_c) / (n * rate_sq);
}

/* problems.cpp:54-76 (validate_params :91-94 first) */
int mgo_exprate_sample_pair(double target_mean, int32_t samples, mgo_mt64* g, double rate_now,
                            double rate_prev, double* prop, double* diff, double* ssn) {
  if (!(rate_now > 0.0) || !(rate_prev > 0.0)) return MG_EDOMAIN;
  double sum_c = 0.0, sum_c_sq = 0.0;
  for (int32_t k = 0; k < samples; ++k) {
    const double c = -log(mgo_uniform_pos(g));
    sum_c += c;
    sum_c_sq += c * c;
  }
  *prop = mgo_exprate_gradient_from_batch(target_mean, samples, rate_now, sum_c, sum_c_sq);
  if (rate_now == rate_prev) {
    *diff = 0.0;
    *ssn = 0.0;
  } else {
    *diff = *prop - mgo_exprate_gradient_from_batch(target_mean, samples, rate_prev, sum_c, sum_c_sq);
    *ssn = (rate_now - rate_prev) * (rate_now - rate_prev);
  }
  return 0;
}

/* problems.cpp:110-139 */
double mgo_multnoise_sample_pair(int32_t dim, double sigma, int32_t samples,
                                 const double* target, mgo_mt64* g, const double* now,
                                 const double* prev, double* prop, double* diff) {
  const size_t draws = (size_t)dim * (size_t)samples;
  double* u = (double*)malloc(draws * sizeof(double));
  double* f = (double*)calloc((size_t)dim, sizeof(double));
  for (size_t k = 0; k < draws; ++k) u[k] = mgo_uniform(g);
  for (int32_t s = 0; s < samples; ++s)
    for (int32_t j = 0; j < dim; ++j)
      f[j] += 1.0 + sigma * (2.0 * u[(size_t)s * dim + j] - 1.0);
  for (int32_t j = 0; j < dim; ++j) f[j] = f[j] / (double)samples;
  int same = 1;
  for (int32_t j = 0; j < dim; ++j) same &= (now[j] == prev[j]);
  double ssn = 0.0;
  for (int32_t j = 0; j < dim; ++j) {
    prop[j] = (now[j] - target[j]) * f[j];
    if (same) {
      diff[j] = 0.0;
    } else {
      const double d = now[j] - prev[j];
      diff[j] = d * f[j];
      ssn += d * d;
    }
  }
  free(u);
  free(f);
  return same ? 0.0 : ssn;
}

/* ---------------------------------------------------------- run_single */

int mgo_problem_dim(const mg_experiment_config* cfg) {
  switch (cfg->problem) {
    case MG_EXP_RATE: return 1;
    case MG_MULT_NOISE: return cfg->dim;
    case MG_MINI_RENDER: return cfg->pixel_count;
  }
  return -1;
}

typedef struct problem_state {
  int kind;
  int dim;
  int64_t draws_per_sample;
  double* target; /* truth: exp-rate 1/target_mean, mult-noise target, mini-render T */
  double* exponents;
  double* init;
} problem_state;

static int problem_init(const mg_experiment_config* cfg, problem_state* p) {
  memset(p, 0, sizeof(*p));
  p->kind = cfg->problem;
  p->dim = mgo_problem_dim(cfg);
  if (p->dim < 1) return MG_EINVAL;
  p->target = (double*)calloc((size_t)p->dim, sizeof(double));
  p->init = (double*)calloc((size_t)p->dim, sizeof(double));
  switch (p->kind) {
    case MG_EXP_RATE: /* problems.cpp:30-42 */
      if (!(cfg->target_mean > 0.0) || cfg->samples_per_iter < 2 || !(cfg->rate_init > 0.0))
        return MG_EINVAL;
      p->target[0] = 1.0 / cfg->target_mean;
      p->init[0] = cfg->rate_init;
      p->draws_per_sample = cfg->samples_per_iter;
      break;
    case MG_MULT_NOISE: /* problems.cpp:99-108, harness.cpp:71-73 (target 0) */
      if (cfg->sigma < 0.0 || cfg->samples_per_iter < 1) return MG_EINVAL;
      for (int j = 0; j < p->dim; ++j) p->init[j] = p->target[j] + 2.0;
      p->draws_per_sample = (int64_t)cfg->samples_per_iter * p->dim;
      break;
    case MG_MINI_RENDER: /* problems.cpp:162-175 */
      if (cfg->spp < 2 || !(cfg->exponent_max >= 0.0)) return MG_EINVAL;
      p->exponents = (double*)calloc((size_t)p->dim, sizeof(double));
      mgo_minirender_generate(p->dim, cfg->problem_seed, cfg->exponent_max, p->exponents, p->target);
      for (int j = 0; j < p->dim; ++j) p->init[j] = cfg->albedo_init;
      p->draws_per_sample = (int64_t)cfg->pixel_count * cfg->spp;
      break;
    default:
      return MG_EINVAL;
  }
  return 0;
}

static void problem_free(problem_state* p) {
  free(p->target);
  free(p->exponents);
  free(p->init);
}

/* returns 0 or MG_EDOMAIN; fills prop/diff, returns ssn via *ssn */
static int problem_sample(const mg_experiment_config* cfg, const problem_state* p, mgo_mt64* g,
                          const double* now, const double* prev, double* prop, double* diff,
                          double* ssn) {
  switch (p->kind) {
    case MG_EXP_RATE:
      return mgo_exprate_sample_pair(cfg->target_mean, cfg->samples_per_iter, g, now[0], prev[0],
                                     prop, diff, ssn);
    case MG_MULT_NOISE:
      *ssn = mgo_multnoise_sample_pair(p->dim, cfg->sigma, cfg->samples_per_iter, p->target, g, now,
                                       prev, prop, diff);
      return 0;
    default:
      *ssn = mgo_minirender_sample_pair(p->dim, cfg->spp, p->exponents, p->target, g, now, prev,
                                        prop, diff);
      return 0;
  }
}

/* problems.cpp:84-87, :146-149, :223-226 */
static double problem_loss(const problem_state* p, const mg_experiment_config* cfg,
                           const double* x) {
  if (p->kind == MG_EXP_RATE) {
    const double err = 1.0 / x[0] - cfg->target_mean;
    return err * err;
  }
  double s = 0.0;
  for (int j = 0; j < p->dim; ++j) {
    const double d = x[j] - p->target[j];
    s += d * d;
  }
  return p->kind == MG_MULT_NOISE ? 0.5 * s : s;
}

/* problems.cpp:78-82, :141-144, :219-222 */
static void problem_true_grad(const problem_state* p, const mg_experiment_config* cfg,
                              const double* x, double* g) {
  if (p->kind == MG_EXP_RATE) {
    const double r = x[0];
    g[0] = (2.0 * (1.0 / r - cfg->target_mean)) * (-1.0 / (r * r));
    return;
  }
  for (int j = 0; j < p->dim; ++j) {
    const double d = x[j] - p->target[j];
    g[j] = p->kind == MG_MULT_NOISE ? d : 2.0 * d;
  }
}

/* problems.cpp:89, :228 (mult-noise: identity) */
static void problem_project(const problem_state* p, double* x) {
  if (p->kind == MG_EXP_RATE) {
    x[0] = (x[0] < 1e-4) ? 1e-4 : x[0];
  } else if (p->kind == MG_MINI_RENDER) {
    for (int j = 0; j < p->dim; ++j) x[j] = (x[j] < 0.0) ? 0.0 : x[j];
  }
}

/* TrajectorySchedule::at (problems.hpp:207-215), from = init, to = truth */
static void schedule_at(const mg_experiment_config* cfg, const problem_state* p, int i,
                        double* out) {
  const int horizon = cfg->iterations;
  int clamped = i < horizon - 1 ? i : horizon - 1;
  if (clamped < 0) clamped = 0;
  if (cfg->trajectory == MG_TRAJ_SCRIPTED_LINEAR) {
    const double f = horizon <= 1 ? 1.0 : (double)clamped / (double)(horizon - 1);
    for (int j = 0; j < p->dim; ++j) out[j] = p->init[j] + (p->target[j] - p->init[j]) * f;
  } else {
    const double e = exp(-cfg->traj_rate * (double)clamped);
    for (int j = 0; j < p->dim; ++j) out[j] = p->target[j] + (p->init[j] - p->target[j]) * e;
  }
}

int mg_config_validate_oracle(const mg_experiment_config* c); /* below */

int mg_config_validate_oracle(const mg_experiment_config* c) {
  /* harness.cpp:42-66 */
  if (c->problem < 0 || c->problem > 2) return MG_EINVAL;
  if (c->optimizer < 0 || c->optimizer > 1) return MG_EINVAL;
  if (c->trajectory < 0 || c->trajectory > 2) return MG_EINVAL;
  if (c->diff_norm < 0 || c->diff_norm > 1) return MG_EINVAL;
  if (c->iterations < 1 || c->replicates < 1) return MG_EINVAL;
  if (!(c->lr > 0.0)) return MG_EINVAL;
  if (!(c->beta_f >= 0.0 && c->beta_f < 1.0)) return MG_EINVAL;
  if (!(c->beta_delta >= 0.0 && c->beta_delta < 1.0)) return MG_EINVAL;
  if (!(c->beta1 >= 0.0 && c->beta1 < 1.0)) return MG_EINVAL;
  if (!(c->beta2 >= 0.0 && c->beta2 < 1.0)) return MG_EINVAL;
  if (c->coord < 0) return MG_EINVAL;
  if (c->non_zero_centred) return MG_EINVAL;
  return 0;
}

typedef struct iter_out {
  double loss, ssn;
  const double *params, *prop, *diff, *mean_est, *var_est, *alpha, *delta, *true_grad;
} iter_out;

typedef void (*record_fn)(void* ctx, int i, const iter_out* o, int dim);

/* harness.cpp:90-200 */
static int run_single_impl(const mg_experiment_config* cfg, int32_t replicate, mg_run_record* rec,
                           record_fn record, void* rctx, double* final_params) {
  int st = mg_config_validate_oracle(cfg);
  if (st) return st;
  problem_state p;
  st = problem_init(cfg, &p);
  if (st) {
    problem_free(&p);
    return st;
  }
  const int d = p.dim;
  if (cfg->coord >= d) {
    problem_free(&p);
    return MG_EINVAL;
  }
  mgo_mt64 rng;
  mgo_rng_stream(&rng, cfg->seed, (uint64_t)replicate);
  const int scripted = cfg->trajectory != MG_TRAJ_OPTIMISE;
  const int use_meta = cfg->optimizer == MG_OPT_META;
  const size_t vb = (size_t)d * sizeof(double);
  double* params = malloc(vb);
  double* prev = malloc(vb);
  double* prop = malloc(vb);
  double* diff = malloc(vb);
  double* iprop = malloc(vb);
  double* idiff = malloc(vb);
  double* m2p = calloc((size_t)d, sizeof(double));
  double* m2d = calloc((size_t)d, sizeof(double));
  double* mean = calloc((size_t)d, sizeof(double));
  double* var = calloc((size_t)d, sizeof(double));
  double* ap = calloc((size_t)d, sizeof(double));
  double* am = calloc((size_t)d, sizeof(double));
  double* av = calloc((size_t)d, sizeof(double));
  double* delta = malloc(vb);
  double* mest = malloc(vb);
  double* vest = malloc(vb);
  double* var_diff = malloc(vb);
  double* tg = malloc(vb);
  double* xs = malloc(vb);
  if (scripted)
    schedule_at(cfg, &p, 0, params);
  else
    memcpy(params, p.init, vb);
  memcpy(prev, params, vb);
  double pf_pow = 1.0, pd_pow = 1.0;
  int64_t pf_cnt = 0, pd_cnt = 0;
  mg_adam_scalars as = {cfg->lr, cfg->beta1, cfg->beta2, cfg->adam_eps, 1.0, 1.0, 0};
  int meta_first = 1;
  memset(rec, 0, sizeof(*rec));
  rec->status = 0;
  int err = 0;
  for (int i = 0; i < cfg->iterations; ++i) {
    int finite = 1;
    for (int j = 0; j < d; ++j) finite &= isfinite(params[j]) ? 1 : 0;
    if (!finite) { /* :116-119 */
      rec->status = 2;
      break;
    }
    double ssn = 0.0;
    st = problem_sample(cfg, &p, &rng, params, use_meta ? prev : params, prop, diff, &ssn);
    if (st == MG_EDOMAIN) { /* :125-128 */
      rec->status = 2;
      break;
    }
    int same = 1;
    for (int j = 0; j < d; ++j) same &= (params[j] == prev[j]);
    const int two_point = use_meta && !same; /* :129 */
    rec->draws_used += p.draws_per_sample;
    rec->evals_used += p.draws_per_sample * (two_point ? 2 : 1);
    const double* alpha_rec = NULL;
    if (use_meta) {
      const double* vp = prop;
      const double* vd = diff;
      double vssn = ssn;
      if (cfg->independent_variance_samples) { /* :137-142 */
        st = problem_sample(cfg, &p, &rng, params, prev, iprop, idiff, &vssn);
        if (st == MG_EDOMAIN) {
          rec->status = 2;
          break;
        }
        rec->draws_used += p.draws_per_sample;
        rec->evals_used += p.draws_per_sample * (two_point ? 2 : 1);
        vp = iprop;
        vd = idiff;
      }
      mgo_moment2_step(d, cfg->beta_f, &pf_pow, &pf_cnt, m2p, vp); /* :144 */
      if (cfg->diff_norm == MG_DIFF_NORM_PER_PARAM) {            /* :146-151 */
        for (int j = 0; j < d; ++j) {
          const double cs = fabs(params[j] - prev[j]);
          xs[j] = cs; /* coord_step */
        }
        if (vssn > 0.0) {
          double* x = malloc(vb);
          for (int j = 0; j < d; ++j) x[j] = vd[j] / ((xs[j] < 1e-150) ? 1e-150 : xs[j]);
          mgo_moment2_step(d, cfg->beta_delta, &pd_pow, &pd_cnt, m2d, x);
          free(x);
        }
        for (int j = 0; j < d; ++j) var_diff[j] = pd_cnt > 0 ? m2d[j] * (xs[j] * xs[j]) : 0.0;
      } else { /* :153-157 */
        if (vssn > 0.0) {
          double* x = malloc(vb);
          const double s = sqrt(vssn);
          for (int j = 0; j < d; ++j) x[j] = vd[j] / s;
          mgo_moment2_step(d, cfg->beta_delta, &pd_pow, &pd_cnt, m2d, x);
          free(x);
        }
        for (int j = 0; j < d; ++j) var_diff[j] = pd_cnt > 0 ? m2d[j] * ssn : 0.0;
      }
      st = mgo_meta_step(d, cfg->lr, cfg->eps_step, cfg->eps_alpha, !cfg->no_alpha_clip, meta_first,
                         mean, var, ap, prop, diff, m2p, var_diff, delta); /* :160 */
      meta_first = 0;
      if (st) {
        err = st;
        break;
      }
      memcpy(mest, mean, vb);
      memcpy(vest, var, vb);
      alpha_rec = ap;
    } else { /* :165-167 */
      mgo_adam_step(d, &as, am, av, prop, delta);
      for (int j = 0; j < d; ++j) {
        mest[j] = am[j] / (1.0 - as.beta1_pow); /* adam.hpp:42 */
        vest[j] = av[j] / (1.0 - as.beta2_pow); /* adam.hpp:43 */
      }
    }
    problem_true_grad(&p, cfg, params, tg);
    iter_out o = {problem_loss(&p, cfg, params), ssn, params, prop, diff, mest, vest, alpha_rec, delta, tg};
    if (record) record(rctx, i, &o, d);
    rec->iterations_run = i + 1;
    memcpy(prev, params, vb); /* :182 */
    if (scripted) {
      schedule_at(cfg, &p, i + 1, params);
    } else {
      for (int j = 0; j < d; ++j) params[j] = params[j] + delta[j];
      problem_project(&p, params);
    }
  }
  if (!err && rec->status != 2 && cfg->converge_threshold > 0.0 && rec->iterations_run > 0) {
    /* :191-198: err = ||rec.params.back() - truth|| */
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
      const double e = prev[j] - p.target[j];
      s += e * e;
    }
    if (sqrt(s) < cfg->converge_threshold) rec->status = 1;
  }
  if (final_params) memcpy(final_params, prev, vb); /* last recorded params */
  free(params); free(prev); free(prop); free(diff); free(iprop); free(idiff);
  free(m2p); free(m2d); free(mean); free(var); free(ap); free(am); free(av);
  free(delta); free(mest); free(vest); free(var_diff); free(tg); free(xs);
  problem_free(&p);
  return err;
}

typedef struct full_ctx {
  const mgo_full_record* out;
} full_ctx;

static void put_vec(double* base, int i, int d, const double* v) {
  if (base && v) memcpy(base + (size_t)i * d, v, (size_t)d * sizeof(double));
}

static void record_full(void* c, int i, const iter_out* o, int d) {
  const mgo_full_record* r = ((full_ctx*)c)->out;
  put_vec(r->params, i, d, o->params);
  if (r->loss) r->loss[i] = o->loss;
  put_vec(r->prop, i, d, o->prop);
  put_vec(r->diff, i, d, o->diff);
  if (r->ssn) r->ssn[i] = o->ssn;
  put_vec(r->mean_est, i, d, o->mean_est);
  put_vec(r->var_est, i, d, o->var_est);
  put_vec(r->alpha, i, d, o->alpha);
  put_vec(r->delta, i, d, o->delta);
  put_vec(r->true_grad, i, d, o->true_grad);
}

int mgo_run_single(const mg_experiment_config* cfg, int32_t replicate, mg_run_record* rec,
                   const mgo_full_record* out) {
  full_ctx c = {out};
  return run_single_impl(cfg, replicate, rec, out ? record_full : NULL, &c, NULL);
}

typedef struct series_ctx {
  const mg_run_series* s;
  int32_t stride;
  int coord;
  const double* truth;
  int has_truth;
} series_ctx;

static void record_series(void* c, int i, const iter_out* o, int d) {
  const series_ctx* sc = (const series_ctx*)c;
  const mg_run_series* s = sc->s;
  const int k = sc->coord;
  const size_t at = (size_t)i * (size_t)sc->stride;
  if (s->param_err) {
    double acc = 0.0;
    for (int j = 0; j < d; ++j) {
      const double e = o->params[j] - sc->truth[j];
      acc += e * e;
    }
    s->param_err[at] = sqrt(acc);
  }
  if (s->loss) s->loss[at] = o->loss;
  if (s->prop) s->prop[at] = o->prop[k];
  if (s->diff) s->diff[at] = o->diff[k];
  if (s->grad_est) s->grad_est[at] = o->mean_est[k];
  if (s->est_var) s->est_var[at] = o->var_est[k];
  if (s->alpha) s->alpha[at] = o->alpha ? o->alpha[k] : NAN;
  if (s->delta) s->delta[at] = o->delta[k];
  if (s->true_grad) s->true_grad[at] = o->true_grad[k];
  if (s->step_sq_norm) s->step_sq_norm[at] = o->ssn;
  if (s->param) s->param[at] = o->params[k];
}

int mgo_run_single_series(const mg_experiment_config* cfg, int32_t replicate, mg_run_record* rec,
                          const mg_run_series* series, int32_t stride, double* final_params) {
  problem_state p;
  int st = problem_init(cfg, &p);
  if (st) {
    problem_free(&p);
    return st;
  }
  series_ctx c = {series, stride, cfg->coord, p.target, 1};
  st = run_single_impl(cfg, replicate, rec, record_series, &c, final_params);
  problem_free(&p);
  return st;
}


/* =====================================================================
 * F1 slice: textured quad under a rectangular area light, direct lighting
 * (BASELINE.json configs[0] "PR1 ref").  Not in the reference:
 * this is the repo's own CPU restatement of its own renderer
 * (paper_2309_15676_b200/csrc/quad.cu), the oracle for that kernel.
 * Scene, estimators and fixed-point adjoint accumulation are specified in
 * DESIGN.md §F1.
 * ===================================================================== */

/* pinhole at (0,0,3) looking -z; image plane z=0 */
static const double QS_HALF = 1.2;      /* image plane half-extent at z=0  */
static const double QS_LX0 = -0.5, QS_LX1 = 0.5, QS_LY0 = 0.8, QS_LY1 = 1.4, QS_LZ = 1.5;
static const double QS_FIX = 1099511627776.0; /* 2^40 fixed-point scale */
static const double QS_PI = 3.14159265358979323846;

/* radiance factor K_c = Le_c / pi * G * A for one NEE sample; 0 if the
 * camera ray misses the quad.  Writes the texel index. */
static void qs_sample(int W, int H, int R, int px, int py, const double u[4], int* texel,
                      double K[3], const double Le[3]) {
  const double nx = ((px + u[0]) / W) * 2.0 - 1.0;
  const double ny = 1.0 - ((py + u[1]) / H) * 2.0;
  const double x = QS_HALF * nx, y = QS_HALF * ny; /* hit on z = 0 */
  if (x < -1.0 || x > 1.0 || y < -1.0 || y > 1.0) {
    *texel = -1;
    K[0] = K[1] = K[2] = 0.0;
    return;
  }
  int tx = (int)(((x + 1.0) * 0.5) * R), ty = (int)(((y + 1.0) * 0.5) * R);
  if (tx > R - 1) tx = R - 1;
  if (ty > R - 1) ty = R - 1;
  *texel = ty * R + tx;
  const double lx = QS_LX0 + u[2] * (QS_LX1 - QS_LX0);
  const double ly = QS_LY0 + u[3] * (QS_LY1 - QS_LY0);
  const double wx = lx - x, wy = ly - y, wz = QS_LZ;
  const double d2 = (wx * wx + wy * wy) + wz * wz;
  const double inv = 1.0 / sqrt(d2);
  const double cz = wz * inv; /* cos at the quad (n=+z) == cos at the light (n=-z) */
  const double area = (QS_LX1 - QS_LX0) * (QS_LY1 - QS_LY0);
  const double G = ((cz * cz) / d2) * area;
  for (int c = 0; c < 3; ++c) K[c] = (Le[c] / QS_PI) * G;
}

static void qs_uniforms(uint64_t key, uint32_t pixel, uint32_t it, uint32_t sid, uint32_t st,
                        double u[4]) {
  const uint32_t ctr[4] = {pixel, it, sid, st};
  uint32_t o[4];
  mgo_philox4x32_10(ctr, key, o);
  for (int k = 0; k < 4; ++k) u[k] = (double)o[k] * 0x1.0p-32;
}

/* Expected-image stand-in: spp-sample mean image [3][H*W] of texture tex
 * [3][R*R] (channel-major), Philox stream `st`, iteration word 0xffffffff. */
void mgo_quad_render(int W, int H, int R, const double* tex, const double Le[3], int spp,
                     uint64_t key, uint32_t st, double* img) {
  for (int py = 0; py < H; ++py)
    for (int px = 0; px < W; ++px) {
      double acc[3] = {0.0, 0.0, 0.0};
      const uint32_t pix = (uint32_t)(py * W + px);
      for (int s = 0; s < spp; ++s) {
        double u[4], K[3];
        int t;
        qs_uniforms(key, pix, 0xffffffffu, (uint32_t)s, st, u);
        qs_sample(W, H, R, px, py, u, &t, K, Le);
        if (t < 0) continue;
        for (int c = 0; c < 3; ++c) acc[c] += tex[c * R * R + t] * K[c];
      }
      for (int c = 0; c < 3; ++c) img[(size_t)c * W * H + pix] = acc[c] / (double)spp;
    }
}

static int64_t qs_fix(double v) { return (int64_t)llrint(v * QS_FIX); }

/* One gradient sample pair of the quad problem:
 *   samples A, B (proportional) and C (finite difference) per pixel;
 *   prop[c][t] = sum_p r_A K_B [t_B] + r_B K_A [t_A],   r_X = a[t_X] K_X - I*
 *   diff[c][t] = sum_p dI_C K_A [t_A] + dI_C K_B [t_B], dI_C = (a - a_prev)[t_C] K_C
 * accumulated in 2^-40 fixed point (order independent), returned as double.
 * loss_est = sum_p,c r_A r_B (unbiased for sum (I - I*)^2). */
void mgo_quad_sample_pair(int W, int H, int R, const double Le[3], const double* target_img,
                          const double* now, const double* prev, uint64_t key, uint32_t it,
                          uint32_t st, double* prop, double* diff, double* loss_est) {
  const int T = R * R;
  int64_t* fp = (int64_t*)calloc((size_t)3 * T, sizeof(int64_t));
  int64_t* fd = (int64_t*)calloc((size_t)3 * T, sizeof(int64_t));
  double loss = 0.0;
  for (int py = 0; py < H; ++py)
    for (int px = 0; px < W; ++px) {
      const uint32_t pix = (uint32_t)(py * W + px);
      double uA[4], uB[4], uC[4], KA[3], KB[3], KC[3];
      int tA, tB, tC;
      qs_uniforms(key, pix, it, 0, st, uA);
      qs_uniforms(key, pix, it, 1, st, uB);
      qs_uniforms(key, pix, it, 2, st, uC);
      qs_sample(W, H, R, px, py, uA, &tA, KA, Le);
      qs_sample(W, H, R, px, py, uB, &tB, KB, Le);
      qs_sample(W, H, R, px, py, uC, &tC, KC, Le);
      for (int c = 0; c < 3; ++c) {
        const double Is = target_img[(size_t)c * W * H + pix];
        const double rA = (tA >= 0 ? now[c * T + tA] * KA[c] : 0.0) - Is;
        const double rB = (tB >= 0 ? now[c * T + tB] * KB[c] : 0.0) - Is;
        const double dI = tC >= 0 ? (now[c * T + tC] - prev[c * T + tC]) * KC[c] : 0.0;
        loss += rA * rB;
        if (tB >= 0) {
          fp[c * T + tB] += qs_fix(rA * KB[c]);
          fd[c * T + tB] += qs_fix(dI * KB[c]);
        }
        if (tA >= 0) {
          fp[c * T + tA] += qs_fix(rB * KA[c]);
          fd[c * T + tA] += qs_fix(dI * KA[c]);
        }
      }
    }
  for (int k = 0; k < 3 * T; ++k) {
    prop[k] = (double)fp[k] / QS_FIX;
    diff[k] = (double)fd[k] / QS_FIX;
  }
  *loss_est = loss;
  free(fp);
  free(fd);
}


/* =====================================================================
 * F1 slice 2: helix of spheres (BASELINE.json configs[2]), own renderer.
 * Multi-bounce path tracing (max 4 vertices) with next-event estimation to a
 * rectangular area light, constant environment, diffuse ground plane and a
 * principled-style BSDF (Lambert diffuse + GGX/Schlick/Smith specular) whose
 * 5 global parameters (base RGB, metalness, roughness) are optimised.
 * Directions are sampled independently of the parameters (cosine-weighted,
 * Malley's method with Philox-addressed rejection candidates), so the
 * parameter derivative is forward-mode along the path and the finite
 * difference shares the complete path.  DESIGN.md §F1b.
 * ===================================================================== */

#define HX_MAXV 4
#define HX_NP 5
static const double HX_EPS = 1e-4;
static const double HX_TANH = 0.35;
static const double HX_LY = 4.0;     /* light plane y, x,z in [-1,1], facing -y */
static const double HX_LA = 4.0;     /* light area */

typedef struct hx_scene {
  int W, H, nsph;
  const double* sph; /* [nsph][4]: cx cy cz r */
  double Le[3], env[3], ground[3];
} hx_scene;

static inline double hx_dot(const double a[3], const double b[3]) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

/* closest hit: 0 none, 1 sphere (index *k), 2 ground, 3 light (camera only) */
static int hx_intersect(const hx_scene* S, const double o[3], const double d[3], int want_light,
                        double tmax, double* t_out, int* k_out) {
  double best = tmax;
  int kind = 0, kb = -1;
  for (int k = 0; k < S->nsph; ++k) {
    const double* c = S->sph + 4 * k;
    const double oc[3] = {o[0] - c[0], o[1] - c[1], o[2] - c[2]};
    const double b = hx_dot(oc, d);
    const double cc = hx_dot(oc, oc) - c[3] * c[3];
    const double disc = b * b - cc;
    if (disc < 0.0) continue;
    const double sq = sqrt(disc);
    double t = -b - sq;
    if (t < HX_EPS) t = -b + sq;
    if (t < HX_EPS || t >= best) continue;
    best = t;
    kind = 1;
    kb = k;
  }
  if (d[1] < 0.0) {
    const double t = -o[1] / d[1];
    if (t >= HX_EPS && t < best) {
      best = t;
      kind = 2;
    }
  }
  if (want_light && d[1] > 0.0) {
    const double t = (HX_LY - o[1]) / d[1];
    if (t >= HX_EPS && t < best) {
      const double x = o[0] + t * d[0], z = o[2] + t * d[2];
      if (x >= -1.0 && x <= 1.0 && z >= -1.0 && z <= 1.0) {
        best = t;
        kind = 3;
      }
    }
  }
  *t_out = best;
  *k_out = kb;
  return kind;
}

/* principled BSDF value f[3] and df[3][5] (d/d base_r, base_g, base_b,
 * metal, rough) for unit n, wi, wo with n.wi > 0, n.wo > 0 */
static void hx_bsdf(const double th[HX_NP], const double n[3], const double wi[3],
                    const double wo[3], double f[3], double df[3][HX_NP]) {
  const double metal = th[3], rough = th[4];
  const double alpha = 0.05 + 0.95 * (rough * rough);
  const double a2 = alpha * alpha;
  double h[3] = {wi[0] + wo[0], wi[1] + wo[1], wi[2] + wo[2]};
  const double hl = sqrt(hx_dot(h, h));
  h[0] /= hl; h[1] /= hl; h[2] /= hl;
  const double nh = hx_dot(n, h), ni = hx_dot(n, wi), no = hx_dot(n, wo), ih = hx_dot(wi, h);
  const double den = nh * nh * (a2 - 1.0) + 1.0;
  const double D = a2 / (QS_PI * (den * den));
  const double dD_da2 = (den - 2.0 * a2 * (nh * nh)) / (QS_PI * ((den * den) * den));
  const double si = sqrt(a2 + (1.0 - a2) * (ni * ni));
  const double so = sqrt(a2 + (1.0 - a2) * (no * no));
  const double G1i = (2.0 * ni) / (ni + si), G1o = (2.0 * no) / (no + so);
  const double dG1i = ((-2.0 * ni) / ((ni + si) * (ni + si))) * ((1.0 - ni * ni) / (2.0 * si));
  const double dG1o = ((-2.0 * no) / ((no + so) * (no + so))) * ((1.0 - no * no) / (2.0 * so));
  const double G = G1i * G1o;
  const double dG_da2 = dG1i * G1o + G1i * dG1o;
  const double q = 1.0 - ih;
  const double q5 = ((q * q) * (q * q)) * q;
  const double denom = 4.0 * ni * no;
  const double DG = (D * G) / denom;
  const double dDG_drough = (((dD_da2 * G + D * dG_da2) / denom) * (2.0 * alpha)) * (1.9 * rough);
  for (int c = 0; c < 3; ++c) {
    const double base = th[c];
    const double F0 = 0.04 * (1.0 - metal) + base * metal;
    const double F = F0 + (1.0 - F0) * q5;
    f[c] = ((1.0 - metal) * base) / QS_PI + DG * F;
    for (int k = 0; k < HX_NP; ++k) df[c][k] = 0.0;
    df[c][c] = (1.0 - metal) / QS_PI + DG * (metal * (1.0 - q5));
    df[c][3] = (-base) / QS_PI + DG * ((base - 0.04) * (1.0 - q5));
    df[c][4] = dDG_drough * F;
  }
}

/* Duff et al. orthonormal basis */
static void hx_onb(const double n[3], double T[3], double B[3]) {
  const double sign = copysign(1.0, n[2]);
  const double a = -1.0 / (sign + n[2]);
  const double b = n[0] * n[1] * a;
  T[0] = 1.0 + sign * (n[0] * n[0]) * a; T[1] = sign * b; T[2] = -sign * n[0];
  B[0] = b; B[1] = sign + (n[1] * n[1]) * a; B[2] = -n[1];
}

static void hx_rng(uint64_t key, uint32_t pix, uint32_t it, uint32_t path, uint32_t slot,
                   double u[4]) {
  const uint32_t ctr[4] = {pix, it, path, slot};
  uint32_t o[4];
  mgo_philox4x32_10(ctr, key, o);
  for (int k = 0; k < 4; ++k) u[k] = (double)o[k] * 0x1.0p-32;
}

/* one path for up to two parameter sets; L[s][3], dL[s][3][5] */
static void hx_path(const hx_scene* S, const double th[2][HX_NP], int nsets, int px, int py,
                    uint64_t key, uint32_t it, uint32_t path, double L[2][3],
                    double dL[2][3][HX_NP]) {
  const uint32_t pix = (uint32_t)(py * S->W + px);
  double u[4];
  hx_rng(key, pix, it, path, 0u, u);
  const double sx = ((px + u[0]) / S->W) * 2.0 - 1.0;
  const double sy = 1.0 - ((py + u[1]) / S->H) * 2.0;
  double o[3] = {0.0, 1.0, 6.0};
  double d[3] = {sx * HX_TANH * ((double)S->W / (double)S->H), sy * HX_TANH, -1.0};
  double dl = sqrt(hx_dot(d, d));
  d[0] /= dl; d[1] /= dl; d[2] /= dl;
  double beta[2][3], dbeta[2][3][HX_NP];
  for (int s = 0; s < 2; ++s)
    for (int c = 0; c < 3; ++c) {
      beta[s][c] = 1.0; L[s][c] = 0.0;
      for (int k = 0; k < HX_NP; ++k) { dbeta[s][c][k] = 0.0; dL[s][c][k] = 0.0; }
    }
  for (int v = 0; v < HX_MAXV; ++v) {
    double t;
    int k;
    const int kind = hx_intersect(S, o, d, v == 0, 1e30, &t, &k);
    if (kind == 0) { /* escaped: environment */
      for (int s = 0; s < nsets; ++s)
        for (int c = 0; c < 3; ++c) {
          L[s][c] += beta[s][c] * S->env[c];
          for (int j = 0; j < HX_NP; ++j) dL[s][c][j] += dbeta[s][c][j] * S->env[c];
        }
      return;
    }
    if (kind == 3) { /* camera ray sees the light */
      for (int s = 0; s < nsets; ++s)
        for (int c = 0; c < 3; ++c) L[s][c] += S->Le[c];
      return;
    }
    const double x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
    double n[3];
    if (kind == 1) {
      const double* c = S->sph + 4 * k;
      n[0] = (x[0] - c[0]) / c[3]; n[1] = (x[1] - c[1]) / c[3]; n[2] = (x[2] - c[2]) / c[3];
    } else {
      n[0] = 0.0; n[1] = 1.0; n[2] = 0.0;
    }
    const double wo[3] = {-d[0], -d[1], -d[2]};
    hx_rng(key, pix, it, path, (uint32_t)(v * 256 + 1), u);
    /* next-event estimation */
    const double ly[3] = {-1.0 + 2.0 * u[0], HX_LY, -1.0 + 2.0 * u[1]};
    double w[3] = {ly[0] - x[0], ly[1] - x[1], ly[2] - x[2]};
    const double d2 = hx_dot(w, w);
    const double wl = sqrt(d2);
    w[0] /= wl; w[1] /= wl; w[2] /= wl;
    const double cx = hx_dot(n, w), cl = w[1];
    if (cx > 0.0 && cl > 0.0 && hx_dot(n, wo) > 0.0) {
      double ts;
      int ks;
      if (hx_intersect(S, x, w, 0, wl - HX_EPS, &ts, &ks) == 0) {
        const double gl = ((cx * cl) / d2) * HX_LA;
        for (int s = 0; s < nsets; ++s) {
          double f[3], df[3][HX_NP];
          if (kind == 1) {
            hx_bsdf(th[s], n, w, wo, f, df);
          } else {
            for (int c = 0; c < 3; ++c) {
              f[c] = S->ground[c] / QS_PI;
              for (int j = 0; j < HX_NP; ++j) df[c][j] = 0.0;
            }
          }
          for (int c = 0; c < 3; ++c) {
            const double g = gl * S->Le[c];
            L[s][c] += beta[s][c] * (f[c] * g);
            for (int j = 0; j < HX_NP; ++j)
              dL[s][c][j] += dbeta[s][c][j] * (f[c] * g) + beta[s][c] * (df[c][j] * g);
          }
        }
      }
    }
    if (v == HX_MAXV - 1 || hx_dot(n, wo) <= 0.0) return;
    /* cosine-weighted bounce: Malley, rejection in the unit disk */
    double dx = 0.0, dy = 0.0;
    int got = 0;
    for (uint32_t j = 0; !got && j < 64; ++j) {
      double c4[4];
      if (j == 0) {
        c4[0] = u[2]; c4[1] = u[3]; c4[2] = 2.0; c4[3] = 2.0;
      } else {
        hx_rng(key, pix, it, path, (uint32_t)(v * 256 + 1 + j), c4);
      }
      for (int m = 0; m < 4 && !got; m += 2) {
        const double a = 2.0 * c4[m] - 1.0, b = 2.0 * c4[m + 1] - 1.0;
        if (c4[m] <= 1.0 && a * a + b * b < 1.0) { dx = a; dy = b; got = 1; }
      }
    }
    const double dz = sqrt(fmax(0.0, 1.0 - (dx * dx + dy * dy)));
    double T[3], Bv[3];
    hx_onb(n, T, Bv);
    const double wi[3] = {(dx * T[0] + dy * Bv[0]) + dz * n[0], (dx * T[1] + dy * Bv[1]) + dz * n[1],
                          (dx * T[2] + dy * Bv[2]) + dz * n[2]};
    if (dz <= 0.0) return;
    for (int s = 0; s < nsets; ++s) {
      double f[3], df[3][HX_NP];
      if (kind == 1) {
        hx_bsdf(th[s], n, wi, wo, f, df);
      } else {
        for (int c = 0; c < 3; ++c) {
          f[c] = S->ground[c] / QS_PI;
          for (int j = 0; j < HX_NP; ++j) df[c][j] = 0.0;
        }
      }
      for (int c = 0; c < 3; ++c) {
        const double wgt = f[c] * QS_PI; /* f cos / (cos / pi) */
        for (int j = 0; j < HX_NP; ++j)
          dbeta[s][c][j] = dbeta[s][c][j] * wgt + beta[s][c] * (df[c][j] * QS_PI);
        beta[s][c] = beta[s][c] * wgt;
      }
    }
    o[0] = x[0]; o[1] = x[1]; o[2] = x[2];
    d[0] = wi[0]; d[1] = wi[1]; d[2] = wi[2];
  }
}

void mgo_helix_render(int W, int H, int nsph, const double* sph, const double Le[3],
                      const double env[3], const double ground[3], const double th[HX_NP],
                      int spp, uint64_t key, double* img) {
  hx_scene S = {W, H, nsph, sph, {Le[0], Le[1], Le[2]}, {env[0], env[1], env[2]},
                {ground[0], ground[1], ground[2]}};
  double t2[2][HX_NP];
  for (int k = 0; k < HX_NP; ++k) t2[0][k] = t2[1][k] = th[k];
  for (int py = 0; py < H; ++py)
    for (int px = 0; px < W; ++px) {
      double acc[3] = {0.0, 0.0, 0.0};
      for (int s = 0; s < spp; ++s) {
        double L[2][3], dL[2][3][HX_NP];
        hx_path(&S, (const double(*)[HX_NP])t2, 1, px, py, key, 0xffffffffu, (uint32_t)s, L, dL);
        for (int c = 0; c < 3; ++c) acc[c] += L[0][c];
      }
      for (int c = 0; c < 3; ++c) img[(size_t)c * W * H + (size_t)py * W + px] = acc[c] / spp;
    }
}

/* gradient sample pair for the 5 global parameters:
 *   prop = sum_p,c r_A dI_B + r_B dI_A             (paths A, B at theta_t)
 *   diff = sum_p,c [r_C dI_A + r_A dI_C](theta_t) - [same](theta_{t-1})
 * fixed-point 2^-40 accumulation (order independent). */
void mgo_helix_sample_pair(int W, int H, int nsph, const double* sph, const double Le[3],
                           const double env[3], const double ground[3], const double* target_img,
                           const double now[HX_NP], const double prev[HX_NP], uint64_t key,
                           uint32_t it, double prop[HX_NP], double diff[HX_NP],
                           double* loss_est) {
  hx_scene S = {W, H, nsph, sph, {Le[0], Le[1], Le[2]}, {env[0], env[1], env[2]},
                {ground[0], ground[1], ground[2]}};
  double th[2][HX_NP];
  for (int k = 0; k < HX_NP; ++k) { th[0][k] = now[k]; th[1][k] = prev[k]; }
  int64_t fp[HX_NP] = {0}, fd[HX_NP] = {0};
  double loss = 0.0;
  for (int py = 0; py < H; ++py)
    for (int px = 0; px < W; ++px) {
      double LA[2][3], dA[2][3][HX_NP], LB[2][3], dB[2][3][HX_NP], LC[2][3], dC[2][3][HX_NP];
      hx_path(&S, (const double(*)[HX_NP])th, 2, px, py, key, it, 0u, LA, dA);
      hx_path(&S, (const double(*)[HX_NP])th, 1, px, py, key, it, 1u, LB, dB);
      hx_path(&S, (const double(*)[HX_NP])th, 2, px, py, key, it, 2u, LC, dC);
      const size_t pix = (size_t)py * W + px;
      for (int c = 0; c < 3; ++c) {
        const double Is = target_img[(size_t)c * W * H + pix];
        const double rA = LA[0][c] - Is, rB = LB[0][c] - Is, rC = LC[0][c] - Is;
        const double rA1 = LA[1][c] - Is, rC1 = LC[1][c] - Is;
        loss += rA * rB;
        for (int j = 0; j < HX_NP; ++j) {
          fp[j] += qs_fix(rA * dB[0][c][j]);
          fp[j] += qs_fix(rB * dA[0][c][j]);
          fd[j] += qs_fix((rC * dA[0][c][j] + rA * dC[0][c][j]) -
                          (rC1 * dA[1][c][j] + rA1 * dC[1][c][j]));
        }
      }
    }
  for (int j = 0; j < HX_NP; ++j) {
    prop[j] = (double)fp[j] / QS_FIX;
    diff[j] = (double)fd[j] / QS_FIX;
  }
  *loss_est = loss;
}

/* one path's radiance L[3] and dL/dtheta [3][5] (derivative checks) */
void mgo_helix_path(int W, int H, int nsph, const double* sph, const double Le[3],
                    const double env[3], const double ground[3], const double th[HX_NP], int px,
                    int py, uint64_t key, uint32_t it, uint32_t path, double L[3],
                    double dL[3 * HX_NP]) {
  hx_scene S = {W, H, nsph, sph, {Le[0], Le[1], Le[2]}, {env[0], env[1], env[2]},
                {ground[0], ground[1], ground[2]}};
  double t2[2][HX_NP], L2[2][3], dL2[2][3][HX_NP];
  for (int k = 0; k < HX_NP; ++k) t2[0][k] = t2[1][k] = th[k];
  hx_path(&S, (const double(*)[HX_NP])t2, 1, px, py, key, it, path, L2, dL2);
  for (int c = 0; c < 3; ++c) {
    L[c] = L2[0][c];
    for (int k = 0; k < HX_NP; ++k) dL[c * HX_NP + k] = dL2[0][c][k];
  }
}


/* =====================================================================
 * F1 slice 3: textured triangle-mesh scene (BASELINE.json configs[3]),
 * own renderer.  Objects are triangle meshes (quad, tessellated sphere,
 * seeded displaced sphere), each with its own R x R RGB albedo + roughness
 * texture (nearest texel of the interpolated uv): the parameter vector is
 * [object][channel: base r, g, b, roughness][R*R].  Paths of up to `maxv`
 * vertices with NEE to a rectangular area light (not visible to camera
 * rays) and a constant environment collected by escaping rays.  BSDF: the
 * helix slice's principled BSDF with metalness 0.  Directions are sampled
 * independently of the parameters, so one geometric trace serves both
 * parameter sets of the finite difference.  Parameter gradients are
 * reverse-mode: per vertex the NEE weight, the bounce factor's reciprocal
 * and the roughness derivatives are stored; suffix radiance is accumulated
 * backwards; every (vertex, parameter) contribution is quantised to 2^-40
 * and summed as an integer (order independent).  This oracle intersects by
 * brute force over all triangles (the device uses a BVH; equal results
 * because the closest hit breaks ties on the lower triangle index and the
 * BVH culling is conservative).  DESIGN.md §12.
 * ===================================================================== */

#define MS_MAXV 8
#define MS_REC 18  /* per-triangle record: v0 e1 e2 n(unit) uv0 duv1 duv2 */
static const double MS_TMIN = 1e-9;
static const double MS_OFF = 1e-6;

typedef struct ms_scene {
  int W, H, T, R;
  int nch; /* texture channels: 4 = base rgb, rough (metal 0); 5 = + metal */
  const double* tri;
  const int32_t* obj;
  const double* view; /* cam fwd right up(3 each) tanh ly lx0 lx1 lz0 lz1 Le(3) env(3) maxv */
} ms_scene;

static inline void ms_cross(const double a[3], const double b[3], double r[3]) {
  r[0] = a[1] * b[2] - a[2] * b[1];
  r[1] = a[2] * b[0] - a[0] * b[2];
  r[2] = a[0] * b[1] - a[1] * b[0];
}

/* Moller-Trumbore; 1 on a hit with t > MS_TMIN */
static int ms_tri_hit(const double* r, const double o[3], const double d[3], double* t, double* u,
                      double* v) {
  const double* v0 = r;
  const double* e1 = r + 3;
  const double* e2 = r + 6;
  double p[3], q[3], s[3];
  ms_cross(d, e2, p);
  const double det = hx_dot(e1, p);
  if (det == 0.0) return 0;
  const double inv = 1.0 / det;
  s[0] = o[0] - v0[0]; s[1] = o[1] - v0[1]; s[2] = o[2] - v0[2];
  const double uu = hx_dot(s, p) * inv;
  if (uu < 0.0 || uu > 1.0) return 0;
  ms_cross(s, e1, q);
  const double vv = hx_dot(d, q) * inv;
  if (vv < 0.0 || uu + vv > 1.0) return 0;
  const double tt = hx_dot(e2, q) * inv;
  if (!(tt > MS_TMIN)) return 0;
  *t = tt; *u = uu; *v = vv;
  return 1;
}

int mgo_mesh_closest_hit(int T, const double* tri, const double o[3], const double d[3],
                         double* t_out, double* u_out, double* v_out) {
  double best = INFINITY, bu = 0.0, bv = 0.0;
  int bk = -1;
  for (int k = 0; k < T; ++k) {
    double t, u, v;
    if (ms_tri_hit(tri + (size_t)MS_REC * k, o, d, &t, &u, &v) && t < best) {
      best = t; bu = u; bv = v; bk = k;
    }
  }
  *t_out = best; *u_out = bu; *v_out = bv;
  return bk;
}

static int ms_occluded(const ms_scene* S, const double o[3], const double d[3], double tmax) {
  for (int k = 0; k < S->T; ++k) {
    double t, u, v;
    if (ms_tri_hit(S->tri + (size_t)MS_REC * k, o, d, &t, &u, &v) && t < tmax) return 1;
  }
  return 0;
}

/* BSDF with metalness 0: f_c = base_c / pi + S (S = DG F, channel
 * independent); dS/drough.  Same expressions as hx_bsdf. */
static void ms_bsdf(const double base[3], double rough, const double n[3], const double wi[3],
                    const double wo[3], double f[3], double* dS) {
  const double th[HX_NP] = {base[0], base[1], base[2], 0.0, rough};
  double df[3][HX_NP];
  hx_bsdf(th, n, wi, wo, f, df);
  *dS = df[0][4];
}

typedef struct ms_vert {
  int64_t base;             /* parameter index of (object, channel 0, texel) */
  double A[2][3];           /* beta * Le * G (NEE weight), 0 without NEE */
  double dSn[2];            /* dS/drough at the NEE direction (nch 4) */
  double invfb[2][3];       /* 1 / f(bounce), 0 without a bounce or f == 0 */
  double dSb[2];            /* dS/drough at the bounce direction (nch 4) */
  double C[2][3];           /* NEE contribution */
  double dfn[2][3][3];      /* nch 5: df_c / d(base_c, metal, rough), NEE direction */
  double dfb[2][3][3];      /* nch 5: same at the bounce direction */
} ms_vert;

/* full principled BSDF (nch 5): f[3] and df[c][base_c, metal, rough] */
static void ms_bsdf5(const double base[3], double metal, double rough, const double n[3],
                     const double wi[3], const double wo[3], double f[3], double df3[3][3]) {
  const double th[HX_NP] = {base[0], base[1], base[2], metal, rough};
  double df[3][HX_NP];
  hx_bsdf(th, n, wi, wo, f, df);
  for (int c = 0; c < 3; ++c) {
    df3[c][0] = df[c][c];
    df3[c][1] = df[c][3];
    df3[c][2] = df[c][4];
  }
}

/* One path for nsets parameter sets; L[s][3]; vertices (if vout) and the
 * number of vertices; E[s][3] = environment collected after the last one. */
static int ms_path(const ms_scene* S, const double* const th[2], int nsets, int px, int py,
                   uint64_t key, uint32_t it, uint32_t path, double L[2][3], ms_vert* vout,
                   double E[2][3]) {
  const double* V = S->view;
  const int maxv = (int)V[24];
  const int64_t R2 = (int64_t)S->R * S->R;
  const uint32_t pix = (uint32_t)(py * S->W + px);
  double u[4];
  hx_rng(key, pix, it, path, 0u, u);
  const double sx = ((px + u[0]) / S->W) * 2.0 - 1.0;
  const double sy = 1.0 - ((py + u[1]) / S->H) * 2.0;
  const double ax = sx * (V[12] * ((double)S->W / (double)S->H)), ay = sy * V[12];
  double o[3] = {V[0], V[1], V[2]};
  double d[3];
  for (int i = 0; i < 3; ++i) d[i] = (V[3 + i] + ax * V[6 + i]) + ay * V[9 + i];
  const double dl = sqrt(hx_dot(d, d));
  d[0] /= dl; d[1] /= dl; d[2] /= dl;
  double beta[2][3];
  for (int s = 0; s < 2; ++s)
    for (int c = 0; c < 3; ++c) { beta[s][c] = 1.0; L[s][c] = 0.0; E[s][c] = 0.0; }
  const double la = (V[15] - V[14]) * (V[17] - V[16]);
  int nv = 0;
  for (int v = 0; v < maxv; ++v) {
    double t, bu, bv;
    const int k = mgo_mesh_closest_hit(S->T, S->tri, o, d, &t, &bu, &bv);
    if (k < 0) { /* escaped: environment */
      for (int s = 0; s < nsets; ++s)
        for (int c = 0; c < 3; ++c) {
          E[s][c] = beta[s][c] * V[21 + c];
          L[s][c] += E[s][c];
        }
      return nv;
    }
    const double* r = S->tri + (size_t)MS_REC * k;
    const double x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
    double n[3] = {r[9], r[10], r[11]};
    if (hx_dot(n, d) > 0.0) { n[0] = -n[0]; n[1] = -n[1]; n[2] = -n[2]; }
    const double U = (r[12] + bu * r[14]) + bv * r[16];
    const double W_ = (r[13] + bu * r[15]) + bv * r[17];
    int tx = (int)(U * S->R), ty = (int)(W_ * S->R);
    tx = tx < 0 ? 0 : (tx > S->R - 1 ? S->R - 1 : tx);
    ty = ty < 0 ? 0 : (ty > S->R - 1 ? S->R - 1 : ty);
    const int64_t pbase = (int64_t)S->obj[k] * S->nch * R2 + (int64_t)ty * S->R + tx;
    ms_vert* mv = vout ? &vout[nv] : NULL;
    ms_vert tmp;
    if (!mv) mv = &tmp;
    memset(mv, 0, sizeof(*mv));
    mv->base = pbase;
    ++nv;
    double base[2][3], rough[2], metal[2] = {0.0, 0.0};
    for (int s = 0; s < nsets; ++s) {
      for (int c = 0; c < 3; ++c) base[s][c] = th[s][pbase + c * R2];
      rough[s] = th[s][pbase + 3 * R2];
      if (S->nch == 5) metal[s] = th[s][pbase + 4 * R2];
    }
    const double wo[3] = {-d[0], -d[1], -d[2]};
    const double xo[3] = {x[0] + MS_OFF * n[0], x[1] + MS_OFF * n[1], x[2] + MS_OFF * n[2]};
    hx_rng(key, pix, it, path, (uint32_t)(v * 256 + 1), u);
    /* next-event estimation */
    const double lp[3] = {V[14] + u[0] * (V[15] - V[14]), V[13], V[16] + u[1] * (V[17] - V[16])};
    double w[3] = {lp[0] - x[0], lp[1] - x[1], lp[2] - x[2]};
    const double d2 = hx_dot(w, w);
    const double wl = sqrt(d2);
    w[0] /= wl; w[1] /= wl; w[2] /= wl;
    const double cx = hx_dot(n, w), cl = w[1];
    if (cx > 0.0 && cl > 0.0 && hx_dot(n, wo) > 0.0 && !ms_occluded(S, xo, w, wl - MS_OFF)) {
      const double gl = ((cx * cl) / d2) * la;
      for (int s = 0; s < nsets; ++s) {
        double f[3], dS = 0.0;
        if (S->nch == 5) {
          ms_bsdf5(base[s], metal[s], rough[s], n, w, wo, f, mv->dfn[s]);
        } else {
          ms_bsdf(base[s], rough[s], n, w, wo, f, &dS);
        }
        mv->dSn[s] = dS;
        for (int c = 0; c < 3; ++c) {
          const double A = beta[s][c] * (gl * V[18 + c]);
          mv->A[s][c] = A;
          mv->C[s][c] = A * f[c];
          L[s][c] += mv->C[s][c];
        }
      }
    }
    if (v == maxv - 1 || hx_dot(n, wo) <= 0.0) return nv;
    double dx = 0.0, dy = 0.0;
    int got = 0;
    for (uint32_t j = 0; !got && j < 64; ++j) {
      double c4[4];
      if (j == 0) {
        c4[0] = u[2]; c4[1] = u[3]; c4[2] = 2.0; c4[3] = 2.0;
      } else {
        hx_rng(key, pix, it, path, (uint32_t)(v * 256 + 1 + j), c4);
      }
      for (int m = 0; m < 4 && !got; m += 2) {
        const double a = 2.0 * c4[m] - 1.0, b = 2.0 * c4[m + 1] - 1.0;
        if (c4[m] <= 1.0 && a * a + b * b < 1.0) { dx = a; dy = b; got = 1; }
      }
    }
    const double dz = sqrt(fmax(0.0, 1.0 - (dx * dx + dy * dy)));
    if (dz <= 0.0) return nv;
    double Tb[3], Bb[3];
    hx_onb(n, Tb, Bb);
    const double wi[3] = {(dx * Tb[0] + dy * Bb[0]) + dz * n[0],
                          (dx * Tb[1] + dy * Bb[1]) + dz * n[1],
                          (dx * Tb[2] + dy * Bb[2]) + dz * n[2]};
    for (int s = 0; s < nsets; ++s) {
      double f[3], dS = 0.0;
      if (S->nch == 5) {
        ms_bsdf5(base[s], metal[s], rough[s], n, wi, wo, f, mv->dfb[s]);
      } else {
        ms_bsdf(base[s], rough[s], n, wi, wo, f, &dS);
      }
      mv->dSb[s] = dS;
      for (int c = 0; c < 3; ++c) {
        mv->invfb[s][c] = f[c] != 0.0 ? 1.0 / f[c] : 0.0;
        beta[s][c] = beta[s][c] * (f[c] * QS_PI);
      }
    }
    o[0] = xo[0]; o[1] = xo[1]; o[2] = xo[2];
    d[0] = wi[0]; d[1] = wi[1]; d[2] = wi[2];
  }
  return nv;
}

/* adjoint of one stored path for set s with channel weights w[3] */
static void ms_scatter(const ms_vert* vs, int nv, const double E[3], int s, const double w[3],
                       int64_t R2, int64_t* acc, int nch) {
  double Q[3] = {E[0], E[1], E[2]};
  for (int v = nv - 1; v >= 0 && nch == 5; --v) {
    const ms_vert* m = &vs[v];
    double gm = 0.0, gr = 0.0;
    for (int c = 0; c < 3; ++c) {
      const double fb = m->invfb[s][c];
      const double gb = w[c] * (m->A[s][c] * m->dfn[s][c][0] + Q[c] * (fb * m->dfb[s][c][0]));
      acc[m->base + c * R2] += qs_fix(gb);
      gm += w[c] * (m->A[s][c] * m->dfn[s][c][1] + Q[c] * (fb * m->dfb[s][c][1]));
      gr += w[c] * (m->A[s][c] * m->dfn[s][c][2] + Q[c] * (fb * m->dfb[s][c][2]));
    }
    acc[m->base + 3 * R2] += qs_fix(gr);
    acc[m->base + 4 * R2] += qs_fix(gm);
    for (int c = 0; c < 3; ++c) Q[c] = Q[c] + m->C[s][c];
  }
  for (int v = nv - 1; v >= 0 && nch == 4; --v) {
    const ms_vert* m = &vs[v];
    double gr = 0.0;
    for (int c = 0; c < 3; ++c) {
      const double gb = w[c] * ((m->A[s][c] / QS_PI) + Q[c] * (m->invfb[s][c] / QS_PI));
      acc[m->base + c * R2] += qs_fix(gb);
      gr += w[c] * (m->A[s][c] * m->dSn[s] + Q[c] * (m->invfb[s][c] * m->dSb[s]));
    }
    acc[m->base + 3 * R2] += qs_fix(gr);
    for (int c = 0; c < 3; ++c) Q[c] = Q[c] + m->C[s][c];
  }
}

void mgo_meshx_render(int W, int H, int T, const double* tri, const int32_t* obj, int nch, int R,
                      const double* view, const double* theta, int spp, uint64_t key,
                      double* img) {
  ms_scene S = {W, H, T, R, nch, tri, obj, view};
  const double* th[2] = {theta, theta};
  for (int py = 0; py < H; ++py)
    for (int px = 0; px < W; ++px) {
      double acc[3] = {0.0, 0.0, 0.0};
      for (int s = 0; s < spp; ++s) {
        double L[2][3], E[2][3];
        ms_path(&S, th, 1, px, py, key, 0xffffffffu, (uint32_t)s, L, NULL, E);
        for (int c = 0; c < 3; ++c) acc[c] += L[0][c];
      }
      for (int c = 0; c < 3; ++c) img[(size_t)c * W * H + (size_t)py * W + px] = acc[c] / spp;
    }
}

/* gradient sample pair with n proportional paths 0..n-1 (path 0 = A, also
 * evaluated at theta_{t-1}) and the FD path C = path n:
 *   prop = 2 / (n (n-1)) sum_j (sum_{i != j} r_i) dI_j          (theta_t)
 *   diff = sum_c 2 r_C dI_A (theta_t) - 2 r_C dI_A (theta_{t-1})
 *   loss = 2 / (n (n-1)) sum_{i < j} r_i r_j
 * (n = 2: prop = r_A dI_B + r_B dI_A, loss = r_A r_B).  prop/diff have
 * nobj * nch * R * R entries. */
void mgo_meshx_sample_pair(int W, int H, int T, const double* tri, const int32_t* obj, int nobj,
                           int nch, int R, const double* view, const double* target_img,
                           const double* now, const double* prev, uint64_t key, uint32_t it,
                           int row0, int row1, int nprop, double* prop, double* diff,
                           double* loss_est) {
  ms_scene S = {W, H, T, R, nch, tri, obj, view};
  const int64_t R2 = (int64_t)R * R, np = (int64_t)nobj * nch * R2;
  int64_t* fp = (int64_t*)calloc((size_t)np, sizeof(int64_t));
  int64_t* fd = (int64_t*)calloc((size_t)np, sizeof(int64_t));
  ms_vert* vs = (ms_vert*)malloc(sizeof(ms_vert) * MS_MAXV * (size_t)nprop);
  const double* th[2] = {now, prev};
  const double scale = 2.0 / (nprop * (nprop - 1.0));
  double loss = 0.0;
  for (int py = row0; py < row1; ++py)
    for (int px = 0; px < W; ++px) {
      double Lp[8][2][3], Ep[8][2][3], LC[2][3], EC[2][3];
      int nv[8];
      for (int j = 0; j < nprop; ++j)
        nv[j] = ms_path(&S, th, j == 0 ? 2 : 1, px, py, key, it, (uint32_t)j, Lp[j],
                        vs + (size_t)MS_MAXV * j, Ep[j]);
      ms_path(&S, th, 2, px, py, key, it, (uint32_t)nprop, LC, NULL, EC);
      const size_t pix = (size_t)py * W + px;
      double r[8][3], wC0[3], wC1[3];
      for (int c = 0; c < 3; ++c) {
        const double Is = target_img[(size_t)c * W * H + pix];
        for (int j = 0; j < nprop; ++j) r[j][c] = Lp[j][0][c] - Is;
        wC0[c] = 2.0 * (LC[0][c] - Is);
        wC1[c] = -2.0 * (LC[1][c] - Is);
        double lp = 0.0;
        for (int i = 0; i < nprop; ++i)
          for (int j = i + 1; j < nprop; ++j) lp += r[i][c] * r[j][c];
        loss += lp * scale;
      }
      for (int j = 0; j < nprop; ++j) {
        double w[3];
        for (int c = 0; c < 3; ++c) {
          double acc = 0.0;
          int first = 1;
          for (int i = 0; i < nprop; ++i) {
            if (i == j) continue;
            acc = first ? r[i][c] : acc + r[i][c];
            first = 0;
          }
          w[c] = acc * scale;
        }
        ms_scatter(vs + (size_t)MS_MAXV * j, nv[j], Ep[j][0], 0, w, R2, fp, nch);
      }
      ms_scatter(vs, nv[0], Ep[0][0], 0, wC0, R2, fd, nch);
      ms_scatter(vs, nv[0], Ep[0][1], 1, wC1, R2, fd, nch);
    }
  for (int64_t k = 0; k < np; ++k) {
    prop[k] = (double)fp[k] / QS_FIX;
    diff[k] = (double)fd[k] / QS_FIX;
  }
  free(vs);
  free(fp);
  free(fd);
  *loss_est = loss;
}

int mgo_meshx_path_radiance(int W, int H, int T, const double* tri, const int32_t* obj, int nch,
                            int R, const double* view, const double* theta, int px, int py,
                            uint64_t key, uint32_t it, uint32_t path, double L_out[3]) {
  ms_scene S = {W, H, T, R, nch, tri, obj, view};
  const double* th[2] = {theta, theta};
  double L[2][3], E[2][3];
  const int nv = ms_path(&S, th, 1, px, py, key, it, path, L, NULL, E);
  for (int c = 0; c < 3; ++c) L_out[c] = L[0][c];
  return nv;
}

void mgo_mesh_render(int W, int H, int T, const double* tri, const int32_t* obj, int R,
                     const double* view, const double* theta, int spp, uint64_t key,
                     double* img) {
  mgo_meshx_render(W, H, T, tri, obj, 4, R, view, theta, spp, key, img);
}

void mgo_mesh_sample_pair(int W, int H, int T, const double* tri, const int32_t* obj, int nobj,
                          int R, const double* view, const double* target_img, const double* now,
                          const double* prev, uint64_t key, uint32_t it, int row0, int row1,
                          double* prop, double* diff, double* loss_est) {
  mgo_meshx_sample_pair(W, H, T, tri, obj, nobj, 4, R, view, target_img, now, prev, key, it, row0,
                        row1, 2, prop, diff, loss_est);
}

int mgo_mesh_path_radiance(int W, int H, int T, const double* tri, const int32_t* obj, int R,
                           const double* view, const double* theta, int px, int py, uint64_t key,
                           uint32_t it, uint32_t path, double L_out[3]) {
  return mgo_meshx_path_radiance(W, H, T, tri, obj, 4, R, view, theta, px, py, key, it, path,
                                 L_out);
}
