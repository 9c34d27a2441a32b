/*
 * mgcuda.h — C-ABI of the B200-native gradient meta-estimation hot path.
 *
 * Drop-in boundary for the reference `metagrad` library (arxiv 2309.15676,
 * /root/reference/proj).  The reference boundary is a C++ value-semantics API
 * (SURVEY.md §8(b)); every entry point below names the reference symbol it
 * replaces (file:line, relative to /root/reference/proj).  INTEGRATION.md shows
 * the C++ adapter (include/mgcuda.hpp) and the ctypes binding a maintainer adds.
 *
 * Conventions
 *   - Every function returns an mg_status; MG_OK == 0.  The reference throws:
 *       std::invalid_argument -> MG_EINVAL   (meta.hpp:99, moment2.hpp:33, harness.cpp:42-66)
 *       std::logic_error      -> MG_ELOGIC   (meta.hpp:101, negative variance)
 *       std::domain_error     -> MG_EDOMAIN  (problems.cpp:93, invalid params)
 *     mg_last_error() returns the message of the last failure on this thread.
 *   - Buffers are DEVICE pointers (cudaMalloc / torch CUDA storage), SoA, one
 *     entry per parameter, element type given by the dtype argument
 *     (MG_F32 = float, MG_F64 = double).  Host-side scalars are always double.
 *   - A context owns one device and one CUDA stream; every call is
 *     asynchronous on that stream unless it returns host data.  A context is
 *     single-threaded: use one per host thread / device.
 *   - No torch types, no C++ types cross this boundary.
 *   - There is NO CPU fallback: on a machine without a usable sm_100 device
 *     mg_ctx_create fails with MG_ECUDA.
 */
#ifndef MGCUDA_H_
#define MGCUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MGCUDA_ABI_VERSION 1

typedef enum mg_status {
  MG_OK = 0,
  MG_EINVAL = 1,   /* std::invalid_argument */
  MG_ELOGIC = 2,   /* std::logic_error */
  MG_EDOMAIN = 3,  /* std::domain_error */
  MG_ECUDA = 4,    /* CUDA runtime failure / no device */
  MG_ENOMEM = 5,
  MG_EUNSUPPORTED = 6
} mg_status;

typedef enum mg_dtype { MG_F32 = 0, MG_F64 = 1 } mg_dtype;

/* ExperimentConfig (harness.hpp:18-67).  Strings become enums. */
typedef enum mg_problem_kind { MG_EXP_RATE = 0, MG_MULT_NOISE = 1, MG_MINI_RENDER = 2 } mg_problem_kind;
typedef enum mg_optimizer_kind { MG_OPT_META = 0, MG_OPT_ADAM = 1 } mg_optimizer_kind;
typedef enum mg_trajectory_kind {
  MG_TRAJ_OPTIMISE = 0,
  MG_TRAJ_SCRIPTED_LINEAR = 1,
  MG_TRAJ_SCRIPTED_EXP = 2
} mg_trajectory_kind;
typedef enum mg_diff_norm_kind { MG_DIFF_NORM_GLOBAL = 0, MG_DIFF_NORM_PER_PARAM = 1 } mg_diff_norm_kind;
typedef enum mg_rng_kind {
  MG_RNG_MT64 = 0,   /* bit-exact std::mt19937_64 streams (rng.hpp:23-36) */
  MG_RNG_PHILOX = 1  /* counter-based Philox4x32-10, statistically equivalent */
} mg_rng_kind;

typedef struct mg_experiment_config {
  int32_t problem;     /* mg_problem_kind   (harness.hpp:19) */
  int32_t optimizer;   /* mg_optimizer_kind (harness.hpp:20) */
  int32_t iterations;  /* harness.hpp:21 */
  int32_t replicates;  /* harness.hpp:22 */
  uint64_t seed;       /* harness.hpp:23 */
  double lr, beta_f, beta_delta, beta1, beta2, eps_step, eps_alpha, adam_eps; /* :26-33 */
  int32_t dim;              /* mult-noise :36 */
  int32_t samples_per_iter; /* :38 */
  double sigma;             /* :37 */
  double target_mean;       /* :39 */
  double rate_init;         /* :40 */
  int32_t pixel_count;      /* :41 */
  int32_t spp;              /* :42 */
  uint64_t problem_seed;    /* :43 */
  double albedo_init;       /* :44 */
  double exponent_max;      /* :45 */
  int32_t trajectory;       /* mg_trajectory_kind :48 */
  int32_t diff_norm;        /* mg_diff_norm_kind :57 */
  double traj_rate;         /* :49 */
  int32_t no_alpha_clip;                /* :52 */
  int32_t independent_variance_samples; /* :53 */
  int32_t non_zero_centred;             /* :54 (reserved; rejected) */
  int32_t coord;                        /* :60 */
  double converge_threshold;            /* :61 */
  /* B200-only knobs (not in the reference) */
  int32_t dtype;    /* mg_dtype of the device state/arithmetic; MG_F64 = parity mode */
  int32_t rng;      /* mg_rng_kind */
} mg_experiment_config;

/* Fills the reference defaults (harness.hpp:18-67). */
void mg_config_defaults(mg_experiment_config* cfg);
/* ExperimentConfig::validate (harness.cpp:42-66): MG_EINVAL + message. */
int mg_config_validate(const mg_experiment_config* cfg);

const char* mg_last_error(void);
int mg_abi_version(void);
/* Process-wide tuning switches (tests/benchmarks; unknown names -> MG_EINVAL):
 *   "disable_tma" = 1          mg_meta_update / mg_adam_update on the
 *                              register-streaming kernels instead of the TMA
 *                              bulk-copy pipelines
 *   "tma_variant"  -1 | 0..9   schedule of the TMA meta update (-1 default)
 *   "render_fast" = 0          fp32 mini-render on the IEEE kernel instead of
 *                              the TMA-fed fast one (render_fast.cu)
 *   "render_fast_variant"      -1 | 0..16: the fast kernel's schedule
 *   "cluster_runner" = 0       few-replicate mini-render runs on the
 *                              one-CTA-per-replicate runner
 *   "mesh_persistent"          -1 (auto) | 0..3: bit 0 persistent fp32 isect,
 *                              bit 1 persistent fp32 shadow traversal
 *   "mesh_bvh8" = 1            the persistent traversals walk an eight-wide
 *                              BVH (measured slower; off by default)
 *   "mesh_smem_stack"          1 (default): persistent BVH4 traversal stack in
 *                              shared memory; 0: local memory + top nodes staged
 *   "mesh_qnodes"              1 (default): that traversal reads 64-byte nodes
 *                              with 8-bit quantised child boxes; 0: fp32 nodes
 *   "mesh_scatter_aggregate"=1 warp-aggregated mesh adjoint scatter (measured
 *                              slower at configs[3]/[4]; off by default)
 *   "helix_split" = 0          configs[2] sample pair in one kernel (whole
 *                              pixels per thread) instead of path / combine
 *   "pool_keep_bytes" = n      bytes the default stream-ordered memory pool
 *                              keeps mapped across synchronisations (runner
 *                              workspaces; default 512 MiB, CUDA's own is 0)
 *   "render_vec", "bvh_leaf_size", "mesh_megakernel": see DESIGN.md */
int mg_set_option(const char* name, int64_t value);

/* ---------------------------------------------------------------- context */
typedef struct mg_ctx mg_ctx;
/* stream: a cudaStream_t to adopt (not owned; pass cudaStreamLegacy, i.e.
 * (void*)1, for the legacy default stream), or NULL to create a private
 * non-blocking stream. */
int mg_ctx_create(int device, void* stream, mg_ctx** out);
int mg_ctx_destroy(mg_ctx* ctx);
int mg_ctx_synchronize(mg_ctx* ctx);
/* Probe (tools/s1_producer_probe.py): the cluster runner's mt19937_64
 * producer alone, one CTA streaming the `total` raw (untempered) engine state
 * words behind Rng::stream(seed, rep)'s first `total` outputs into out
 * (device u64, viewed as double*: output o = temper(out[o])); progress =
 * device u64. */
int mg_mt_stream_probe(mg_ctx* ctx, uint64_t seed, uint64_t rep, int64_t total, double* out,
                       unsigned long long* progress);
/* Device-check build (libmgcuda_debug.so, MG_DEBUG_CHECKS) only: trips one
 * device assert on purpose -> MG_ECUDA; release builds -> MG_EUNSUPPORTED. */
int mg_debug_selftest(mg_ctx* ctx);
void* mg_ctx_stream(mg_ctx* ctx);
/* Device-side iteration index for graph-replayable optimisation loops: while
 * set (non-NULL), the quad and helix sample-pair kernels launched on ctx use
 * iteration + *dev_counter as their Philox iteration counter, and
 * mg_iteration_offset_add (a one-thread kernel on ctx's stream) advances it,
 * so a captured block of iterations replays with fresh random numbers. */
int mg_ctx_set_iteration_offset(mg_ctx* ctx, const uint32_t* dev_counter);
int mg_iteration_offset_add(mg_ctx* ctx, uint32_t* dev_counter, uint32_t inc);
/* Number of kernels this context has launched so far (bench gpu_launches). */
int64_t mg_ctx_launch_count(mg_ctx* ctx);

/* Device memory helpers so host adapters need nothing but this library.
 * mg_malloc/mg_free are stream-ordered on the context's stream; the copies
 * synchronise the stream; mg_fill writes `value` (cast to dtype) n times. */
int mg_malloc(mg_ctx* ctx, size_t bytes, void** out);
int mg_free(mg_ctx* ctx, void* p);
int mg_copy_to_device(mg_ctx* ctx, void* dst, const void* src, size_t bytes);
int mg_copy_to_host(mg_ctx* ctx, void* dst, const void* src, size_t bytes);
int mg_copy_device(mg_ctx* ctx, void* dst, const void* src, size_t bytes);
/* Page-locked host staging memory (cudaMallocHost) and a stream-ordered
 * copy in any direction (cudaMemcpyDefault; asynchronous w.r.t. the host
 * when the host side is page-locked — pair with mg_ctx_synchronize). */
int mg_host_malloc(size_t bytes, void** out);
int mg_host_free(void* p);
int mg_copy_async(mg_ctx* ctx, void* dst, const void* src, size_t bytes);
int mg_fill(mg_ctx* ctx, int32_t dtype, int64_t n, void* dst, double value);

/* -------------------------------------------------- RNG streams (row A1) */
/* mix64 splitmix64 finaliser (rng.hpp:9-14) — host helper. */
uint64_t mg_mix64(uint64_t x);
/* Replicate stream seed mix64(mix64(seed) ^ (r + 0x51ed2701e35f3a6d)) (rng.hpp:23-25). */
uint64_t mg_stream_seed(uint64_t base_seed, uint64_t replicate);

/* A batch of R independent std::mt19937_64 engines resident on the device
 * (312 x u64 state each, SoA).  seeds[R] are ENGINE seeds (already mixed). */
typedef struct mg_mt64 mg_mt64;
int mg_mt64_create(mg_ctx* ctx, int32_t streams, const uint64_t* host_seeds, mg_mt64** out);
int mg_mt64_destroy(mg_mt64* g);
/* Draws n consecutive outputs from every stream into out[stream][n]:
 * kind 0 = raw u64 (engine_()), 1 = uniform() double (rng.hpp:28),
 * 2 = uniform_pos() double (rng.hpp:31). */
int mg_mt64_draw(mg_ctx* ctx, mg_mt64* g, int64_t n, int32_t kind, void* out);

/* Engine state of stream `stream` in std::mt19937_64's own layout (the 312
 * state words and the position 0..312, as its operator<< writes them), so
 * a host engine (the reference's Rng, rng.hpp:36) can continue on the
 * device and resume on the host bit-exactly. */
int mg_mt64_set_state(mg_ctx* ctx, mg_mt64* g, int32_t stream, const uint64_t* words,
                      int32_t idx);
int mg_mt64_get_state(mg_ctx* ctx, mg_mt64* g, int32_t stream, uint64_t* words, int32_t* idx);

/* GF(2) jump-ahead (Haramoto et al. 2008): advance every stream of g by
 * `distance` draws in O(19937) work, so many engines can produce disjoint
 * segments of ONE replicate's stream bit-exactly.  Streams must sit at a
 * 312-draw block boundary (freshly created, or having drawn a multiple of
 * 312 since) — MG_EINVAL otherwise.  Synchronises the stream. */
int mg_mt64_jump(mg_ctx* ctx, mg_mt64* g, uint64_t distance);
/* `segments` engines positioned at draws c*segment_len (c = 0..segments-1)
 * of the single stream seeded with engine_seed.  With segment_len a multiple
 * of 312, drawing segment_len from every engine yields draws
 * [0, segments*segment_len) of the stream in [engine][draw] order; jumping
 * all by (D - segment_len) then positions them for the next D-draw block. */
int mg_mt64_split(mg_ctx* ctx, uint64_t engine_seed, int32_t segments, uint64_t segment_len,
                  mg_mt64** out);
/* Host helper: g(x) = x^distance mod phi(x) as 312 little-endian words and
 * its degree (phi = characteristic polynomial of mt19937_64, recovered once
 * with Berlekamp-Massey).  No device needed. */
int mg_mt64_jump_polynomial(uint64_t distance, uint64_t* out_words, int32_t* out_deg);

/* ------------------------------------- fused estimator kernels (A8-A12) */
/* Host-owned scalar state of one Moment2 (moment2.hpp:45-47).  The device
 * only ever sees the per-step coefficient w/w_sum computed from it in fp64,
 * exactly as moment2.hpp:35-38 does. */
typedef struct mg_moment2_scalars {
  double decay;
  double decay_pow; /* decay^count by repeated multiplication (moment2.hpp:35) */
  int64_t count;
} mg_moment2_scalars;

/* Moment2::step (moment2.hpp:30-39) on a device vector. */
int mg_moment2_step(mg_ctx* ctx, int32_t dtype, int64_t n, mg_moment2_scalars* s, void* m2,
                    const void* x);

/* MetaEstimator hyper-parameters (meta.hpp:72-75). */
typedef struct mg_meta_params {
  double lr;
  double eps_step;
  double eps_alpha;
  int32_t clip_enabled;
} mg_meta_params;

/* MetaEstimator::step (meta.hpp:90-113) on device buffers: updates mean, var,
 * alpha_prev in place and writes delta.  first_call != 0 performs the lazy
 * initialisation of meta.hpp:92-96 (mean=0, var=0, alpha_prev=-inf) first.
 * Negative var_prop / var_diff -> MG_ELOGIC (meta.hpp:100-101); the check is
 * a device reduction and this call synchronises the stream. */
int mg_meta_step(mg_ctx* ctx, int32_t dtype, int64_t n, const mg_meta_params* p,
                 int32_t first_call, void* mean, void* var, void* alpha_prev, const void* prop,
                 const void* diff, const void* var_prop, const void* var_diff, void* delta);

/* compute_alpha (meta.hpp:38-47), the standalone clipped weight:
 * out = min(vp / (((vp + var_meta) + var_diff) + eps_alpha), 1 / (2 - alpha_prev)).
 * A negative variance input -> MG_ELOGIC (synchronises the stream). */
int mg_compute_alpha(mg_ctx* ctx, int32_t dtype, int64_t n, const void* var_prop,
                     const void* var_meta, const void* var_diff, const void* alpha_prev,
                     double eps_alpha, void* out);

/* out = x * s (op 0: rescale_diff_variance, meta.hpp:51-53) or
 * out = x / s (op 1: Adam::m_hat / v_hat bias correction, adam.hpp:43-44). */
int mg_scalar_op(mg_ctx* ctx, int32_t dtype, int64_t n, const void* x, double s, int32_t op,
                 void* out);

/* Adam::step (adam.hpp:23-37).  b1pow/b2pow/t live on the host like the
 * reference's members (adam.hpp:47-48) and are advanced by this call. */
typedef struct mg_adam_scalars {
  double lr, beta1, beta2, eps;
  double beta1_pow, beta2_pow;
  int64_t t;
} mg_adam_scalars;
int mg_adam_step(mg_ctx* ctx, int32_t dtype, int64_t n, mg_adam_scalars* s, void* m, void* v,
                 const void* grad, void* delta);

/* ---------------------------------------------------------------------------
 * The fused hot-path update: one HBM pass per iteration that does
 *   Moment2(beta_f).step(prop)                         moment2.hpp:30-39, harness.cpp:144
 *   global-norm diff decoupling + Moment2(beta_delta)  harness.cpp:153-157, meta.hpp:51-53
 *   MetaEstimator::step                                meta.hpp:90-113
 *   params += delta; project (max(p, lo) if enabled)   harness.cpp:182-188, problems.cpp:228
 *   sum (p_new - p_old)^2  -> next iteration's step_sq_norm  (problems.cpp:214)
 *   sum (p_new - target)^2 -> loss of the new params         (problems.cpp:225)
 * The step_sq_norm that scales THIS step's diff is read from device memory
 * (written by the previous step's reduction), so consecutive steps run with
 * no host synchronisation and can be captured in a CUDA graph.  The diff-EMA
 * count therefore lives on the device as well (it only advances when
 * step_sq_norm > 0, harness.cpp:153).
 * ------------------------------------------------------------------------- */
typedef struct mg_update_scalars {
  /* Reduced block, written by step t's epilogue for step t+1.  Plain element
   * sums, contiguous, so a sharded step all-reduces them with one SUM. */
  double ssn;       /* sum (p_new - p_old)^2 -> next step_sq_norm (problems.cpp:214) */
  double changed;   /* count of p_new != p_old (problems.cpp:206, "same" test) */
  double loss;      /* sum (p_new - target)^2 (problems.cpp:225), NaN without target */
  double nonfinite; /* count of non-finite p_new (harness.cpp:116) */
  /* Decoupled diff-EMA scalars (moment2.hpp:45-47), advanced on the device:
   * the EMA only steps when step_sq_norm > 0 (harness.cpp:153). */
  double diff_decay_pow;
  int64_t diff_count;
  /* What step t consumed, for recording (harness.cpp:174). */
  double ssn_used;
  /* beta_f^t of Moment2(beta_f) (moment2.hpp:35), advanced on the device by
   * every launch whose args carry prop_pow_advance (or beta_f > 0); read when
   * prop_coef_device. */
  double prop_decay_pow;
} mg_update_scalars;

typedef struct mg_meta_update_args {
  mg_meta_params meta;
  double prop_coef;      /* (1-beta_f)/(1-beta_f^t), host fp64 (moment2.hpp:36-38) */
  double beta_delta;     /* decay of the decoupled diff EMA (harness.hpp:28) */
  int32_t first_step;    /* lazy init of Moment2 / MetaEstimator state (moment2.hpp:31, meta.hpp:92-96) */
  int32_t diff_norm;     /* mg_diff_norm_kind (harness.cpp:146-158) */
  int32_t project;       /* 1: p = max(p, proj_lo) (problems.cpp:228 uses 0.0);
                            2: p = min(max(p, proj_lo), proj_hi) */
  int32_t ssn_from_host; /* 1: step_sq_norm = ssn_host instead of scalars->ssn */
  double proj_lo;
  double ssn_host;
  double proj_hi;
  double beta_f;            /* decay of Moment2(beta_f); see prop_pow_advance */
  int32_t prop_coef_device; /* 1: Moment2(beta_f) coefficient (1-beta_f)/(1-prop_decay_pow)
                               from the device power instead of prop_coef — steps that
                               carry no per-step host scalar, so one captured CUDA graph
                               can be replayed (same bits: same IEEE multiply chain) */
  int32_t prop_pow_advance; /* 1: advance scalars->prop_decay_pow *= beta_f on the device
                               (every step of a run that uses prop_coef_device).  Legacy:
                               beta_f > 0 also advances.  beta_f = 0 is a valid decay
                               (coefficient 1, moment2.hpp:36-38); with prop_coef_device it
                               needs this flag, else MG_EINVAL. */
} mg_meta_update_args;

/* Optional side inputs/outputs of the fused update.  Any may be NULL. */
typedef struct mg_meta_extras {
  const void* vprop;       /* independent variance pair (harness.cpp:137-142) */
  const void* vdiff;
  const void* params_prev; /* pi_{t-1}, per-param diff norm only (harness.cpp:147) */
  const void* target;      /* for the fused loss (problems.cpp:225) */
  void* delta_out;         /* the step delta (harness.cpp:160) */
} mg_meta_extras;

/* One fused meta-estimator iteration over n parameters.
 *   prop, diff            : this iteration's gradient sample pair (read)
 *   m2_prop, m2_diff      : Moment2 states (read+write)
 *   mean, var, alpha_prev : MetaEstimator state (read+write)
 *   params_in             : pi_t (read);  params_out: pi_{t+1} (write; may == params_in)
 *   scalars               : device mg_update_scalars (read ssn/diff state, write next)
 *   x                     : optional extras (NULL for none)
 * The host only supplies prop_coef (a pure function of the iteration count). */
int mg_meta_update(mg_ctx* ctx, int32_t dtype, int64_t n, const mg_meta_update_args* a,
                   const void* prop, const void* diff, void* m2_prop, void* m2_diff, void* mean,
                   void* var, void* alpha_prev, const void* params_in, void* params_out,
                   mg_update_scalars* scalars, const mg_meta_extras* x);

/* mg_meta_update whose sample pair is the texel-interleaved 2^-40
 * fixed-point accumulator a mesh sample pair leaves behind when called with
 * prop = diff = NULL (mg_meshscene_sample_pair): accum = int64
 * [cells][prop | diff][nch], cells = objects * r2; parameters planar
 * [object][nch][r2], n = cells * nch.  prop_i / diff_i = (double)word / 2^40
 * rounded to dtype — exactly what mg_meshscene_sample_pair would have written
 * — and the accumulator is zeroed, so every element equals the unfused
 * finalize + mg_meta_update (the reductions may sum in another order).  One
 * pass: the planar pair is never stored (16 B less HBM traffic per
 * parameter).  No reference counterpart beyond mg_meta_update's
 * (harness.cpp:144-188); x->vprop / vdiff -> MG_EUNSUPPORTED. */
int mg_meta_update_fixed(mg_ctx* ctx, int32_t dtype, int64_t cells, int32_t nch, int32_t r2,
                         const mg_meta_update_args* a, void* accum, void* m2_prop, void* m2_diff,
                         void* mean, void* var, void* alpha_prev, const void* params_in,
                         void* params_out, mg_update_scalars* scalars, const mg_meta_extras* x);
/* mg_meta_update_fixed with a touch map: touch_map holds one bit per texel
 * cell (cells / 32 uint32 words, cell c = bit c % 32 of word c / 32; zero
 * before first use) and bit c is set whenever accum's cell c may be
 * non-zero — mg_meshscene_set_touch_map makes the accumulator-keeping sample
 * pair maintain it.  Only the cells whose bit is set are read and zeroed
 * (an untouched cell's pair is exactly 0 either way, so the results are
 * identical to mg_meta_update_fixed) and their bits are cleared; in a large
 * texture set most cells see no path in an iteration, so most of the 32
 * accumulator bytes per parameter are never moved.  touch_map NULL: the same
 * as mg_meta_update_fixed.  A stale set bit only costs its cell's read. */
int mg_meta_update_fixed_touch(mg_ctx* ctx, int32_t dtype, int64_t cells, int32_t nch, int32_t r2,
                               const mg_meta_update_args* a, void* accum, uint32_t* touch_map,
                               void* m2_prop, void* m2_diff, void* mean, void* var,
                               void* alpha_prev, const void* params_in, void* params_out,
                               mg_update_scalars* scalars, const mg_meta_extras* x);

/* Tile-sharded SHARED parameters (configs 4/5 shape), one rank's step as one
 * kernel over peer memory: for the parameter shard [shard_lo, shard_lo +
 * shard_n) it sums the world ranks' partial sample pairs prop_parts[q],
 * diff_parts[q] (device pointers to full-length vectors, local or NVLink
 * peer, summed in rank order 0..world-1), runs the fused meta update on its
 * shard state (m2_prop.. alpha_prev, target: shard-length), and stores the
 * new parameters into params_out[q] + shard_lo for every rank q
 * (all-gather).  params_in is this rank's full current parameter vector.
 * world <= 8.  The caller fences the ranks around the call (e.g. a
 * symmetric-memory barrier) and all-reduces the first 4 scalars. */
int mg_shared_meta_update(mg_ctx* ctx, int32_t dtype, int64_t shard_n, int64_t shard_lo,
                          int32_t world, const mg_meta_update_args* a,
                          const void* const* prop_parts, const void* const* diff_parts,
                          void* const* params_out, const void* params_in, void* m2_prop,
                          void* m2_diff, void* mean, void* var, void* alpha_prev,
                          const void* target, mg_update_scalars* scalars);

/* Fused Adam baseline iteration (adam.hpp:23-37 + harness.cpp:165-166,
 * 182-188): m, v updated, params_out = project(params_in + delta), with the
 * same ssn/loss reductions into scalars. */
int mg_adam_update(mg_ctx* ctx, int32_t dtype, int64_t n, mg_adam_scalars* s, int32_t project,
                   double proj_lo, const void* grad, void* m, void* v, const void* params_in,
                   void* params_out, const void* target, mg_update_scalars* scalars);

/* Device -> host copy of a scalars block (synchronises the stream). */
int mg_scalars_read(mg_ctx* ctx, const mg_update_scalars* dev, mg_update_scalars* host);
int mg_scalars_write(mg_ctx* ctx, mg_update_scalars* dev, const mg_update_scalars* host);

/* ------------------------------------ gradient-sample sources (A2-A7) */
/* MiniRenderProblem (problems.hpp:157-195, problems.cpp:162-228).
 * Construction draws b_j then T_j from Rng(mix64(gen_seed)) on the device
 * (problems.cpp:168-172); out buffers are fp64 [P]. */
int mg_minirender_generate(mg_ctx* ctx, int32_t pixel_count, uint64_t gen_seed, double exponent_max,
                           double* exponents, double* target);

/* MiniRenderProblem::sample_pair (problems.cpp:197-217) for R replicates at
 * once.  Replicate r draws P*spp uniforms from stream r of g (pixel-major,
 * problems.cpp:201-202), then per pixel computes kernel_terms (:177-195) and
 *   prop = 2 a_now cross - 2 T mean_basis,  diff = 2 (a_now - a_prev) cross.
 * now/prev/prop/diff are [R][P] of dtype; exponents/target fp64 [P] shared.
 * ssn_out[R] (fp64, device) receives sum (a_now - a_prev)^2 (0 when equal).
 * If now == prev bitwise for a replicate, diff = 0 and ssn = 0 exactly. */
int mg_minirender_sample_pair(mg_ctx* ctx, int32_t dtype, int32_t replicates, int32_t pixel_count,
                              int32_t spp, const double* exponents, const double* target,
                              mg_mt64* g, const void* now, const void* prev, void* prop, void* diff,
                              double* ssn_out);

/* ExpRateProblem::sample_pair (problems.cpp:54-76), R replicates (dim 1).
 * rate_now/rate_prev/prop/diff/ssn are fp64 [R].  Non-positive rates ->
 * MG_EDOMAIN (synchronises). */
int mg_exprate_sample_pair(mg_ctx* ctx, int32_t replicates, double target_mean,
                           int32_t samples_per_iter, mg_mt64* g, const double* rate_now,
                           const double* rate_prev, double* prop, double* diff, double* ssn);

/* MultNoiseQuadratic::sample_pair (problems.cpp:121-139), R replicates,
 * uniforms sample-major u[s*d+j].  All buffers fp64; target [d] shared,
 * now/prev/prop/diff [R][d], ssn [R]. */
int mg_multnoise_sample_pair(mg_ctx* ctx, int32_t replicates, int32_t dim, double sigma,
                             int32_t samples_per_iter, const double* target, mg_mt64* g,
                             const double* now, const double* prev, double* prop, double* diff,
                             double* ssn);

/* One FUSED mini-render meta iteration over P pixels: sample_pair
 * (problems.cpp:197-217) at (pi_t, pi_{t-1}) on shared draws, then the fused
 * update of mg_meta_update with projection max(p, 0) (problems.cpp:228); the
 * sample pair stays in registers (optionally copied to prop_out/diff_out).
 *   rng_kind MG_RNG_MT64 : uniforms[P*spp] are this iteration's draws of the
 *                          replicate stream (mg_mt64_draw), pixel-major —
 *                          the reference's exact sample stream.
 *   rng_kind MG_RNG_PHILOX: uniform s of pixel j = Philox4x32-10 with
 *                          counter (j, iteration, s/2, stream), key = `key`
 *                          (statistically equivalent scale mode).
 * params_prev_next holds pi_{t-1} on entry and pi_{t+1} on exit.
 * Pixel sharding: a rank owning pixels [lo, lo+P) passes pixel_offset = lo
 * (Philox counters use the global index) and, in mt64 mode, the slice
 * uniforms + lo*spp of the full iteration stream; then all-reduces the
 * first 4 doubles of *scalars (SUM) before the next iteration.
 * exponents/target are dtype arrays [P].  "same" (diff = 0) is taken from
 * scalars->changed == 0, the previous step's reduction. */
typedef struct mg_render_args {
  mg_meta_update_args update; /* meta params, prop_coef, beta_delta, first_step, ssn override */
  int32_t spp;
  int32_t rng_kind;
  uint64_t key;       /* mg_stream_seed(seed, replicate) */
  uint32_t iteration; /* Philox counter word 1 */
  uint32_t stream;    /* Philox counter word 3 (0: main pair, 1: independent pair) */
  uint32_t pixel_offset; /* global index of local pixel 0 (pixel-sharded runs) */
  int32_t record_plus1;  /* 0: prop_out/diff_out (if given) are full [P] arrays;
                            k+1: they are single values and receive local pixel k */
} mg_render_args;

int mg_minirender_meta_iteration(mg_ctx* ctx, int32_t dtype, int64_t P, const mg_render_args* a,
                                 const void* exponents, const void* target,
                                 const double* uniforms, const void* params_now,
                                 void* params_prev_next, void* m2_prop, void* m2_diff, void* mean,
                                 void* var, void* alpha_prev, mg_update_scalars* scalars,
                                 void* prop_out, void* diff_out);

/* ---------------------------------------------------------------------------
 * F1 slice (BASELINE.json configs[0]): path-traced gradient
 * samples of a textured quad under a rectangular area light, direct lighting,
 * Lambertian BSDF, RGB texture R x R (nearest), image W x H.  Not in the
 * reference: scene and estimators are this repo's own
 * (DESIGN.md §F1), checked against oracle/metagrad_oracle.c mgo_quad_*.
 * Textures/gradients are channel-major [3][R*R], images [3][H*W], dtype
 * arrays; Le is the light's RGB radiance (host).  Philox counters
 * (pixel, iteration, sample, stream) with key = replicate seed.
 * ------------------------------------------------------------------------- */
/* spp-sample mean image of texture tex (iteration word 0xffffffff). */
int mg_quad_render(mg_ctx* ctx, int32_t dtype, int32_t W, int32_t H, int32_t R, const double* Le,
                   int32_t spp, uint64_t key, uint32_t stream, const void* tex, void* img);
/* One gradient sample pair: prop/diff [3][R*R] (1 FD + 2 proportional spp
 * per pixel), loss_out (device double) = unbiased estimate of
 * sum (I - I*)^2.  accum: device scratch of 6*R*R int64, zero on first use
 * (left zeroed).  Deterministic (fixed-point adjoint accumulation).
 * Tile sharding: only image rows [row0, row1) contribute (0, H for all);
 * the partial pairs of disjoint tiles sum EXACTLY to the full pair. */
int mg_quad_sample_pair(mg_ctx* ctx, int32_t dtype, int32_t W, int32_t H, int32_t R,
                        const double* Le, const void* target_img, const void* now,
                        const void* prev, uint64_t key, uint32_t iteration, uint32_t stream,
                        int32_t row0, int32_t row1, void* accum, void* prop, void* diff,
                        double* loss_out);

/* F1 slice 2 (BASELINE.json configs[2]): helix of spheres on a diffuse ground
 * plane, rectangular area light (y=4, x,z in [-1,1]) + constant environment,
 * depth-4 path tracing with NEE, principled BSDF with 5 global parameters
 * theta = (base r, g, b, metalness, roughness).
 * spheres: device fp64 [nsph][4] (center, radius), nsph <= 256; Le/env/ground
 * host fp64 RGB triples; theta/now/prev DEVICE dtype 5-vectors (read by the
 * kernel: no host round trip per iteration); images [3][H*W] dtype. */
int mg_helix_render(mg_ctx* ctx, int32_t dtype, int32_t W, int32_t H, int32_t nsph,
                    const double* spheres, const double* Le, const double* env,
                    const double* ground, const void* theta, int32_t spp, uint64_t key,
                    void* img);
/* One gradient sample pair for theta: prop/diff are dtype [5] (device),
 * loss_out device double, accum device scratch of 10 int64 (zero, left zero).
 * Paths A, B (proportional) and C (finite difference, A and C evaluated at
 * theta_now and theta_prev on the same path). */
int mg_helix_sample_pair(mg_ctx* ctx, int32_t dtype, int32_t W, int32_t H, int32_t nsph,
                         const double* spheres, const double* Le, const double* env,
                         const double* ground, const void* target_img, const void* now,
                         const void* prev, uint64_t key, uint32_t iteration, int32_t row0,
                         int32_t row1, void* accum, void* prop, void* diff, double* loss_out);

/* ------------------------ F1 slice 3: textured triangle-mesh scene (configs[3]) */
/* Scene of T triangles (host fp64 records [T][18]: v0, e1 = v1 - v0,
 * e2 = v2 - v0, unit geometric normal, uv0, uv1 - uv0, uv2 - uv0; object id
 * per triangle in [0, nobj)); each object owns an R x R texture of
 * `channels` parameters per texel: 4 = base r, g, b, roughness (metalness
 * 0; configs[3]) or 5 = + metalness (configs[4]): parameters
 * [nobj][channels][R*R].  The BVH is built on the host (binned SAH,
 * breadth-first node order) and uploaded.
 * view[25] = camera position, forward, right, up (3 each), tan(fov_y/2),
 * light plane y, light x0, x1, z0, z1, light radiance rgb, environment rgb,
 * max path vertices (1..8).  DESIGN.md §12; oracle mgo_mesh_*. */
typedef struct mg_mesh_scene mg_mesh_scene;
int mg_meshscene_create(mg_ctx* ctx, int32_t tri_count, const double* tri, const int32_t* obj,
                        int32_t nobj, int32_t tex_res, int32_t channels, mg_mesh_scene** out);
int mg_meshscene_destroy(mg_mesh_scene* s);
int mg_meshscene_info(const mg_mesh_scene* s, int32_t* nodes, int32_t* depth, int64_t* params);
/* Opt-in for optimisation loops that ping-pong their parameter buffers: the
 * caller promises that whenever a sample-pair call's `prev` equals the
 * previous call's `now` pointer, it still holds the values it held then.
 * The shade stage's texel-major copy of that buffer is then reused instead
 * of rebuilt (one relayout per iteration instead of two). */
int mg_meshscene_set_prev_reuse(mg_mesh_scene* s, int32_t enable);
/* touch_map (caller-owned, objects * R^2 / 32 uint32 words rounded up, or
 * NULL to stop): sample pairs that leave their pair in accum (prop = diff =
 * NULL) set the bit of every texel cell they add to, for
 * mg_meta_update_fixed_touch.  The map belongs with ONE accumulator. */
int mg_meshscene_set_touch_map(mg_mesh_scene* s, uint32_t* touch_map);
/* Diagnostics (no reference counterpart): the queue counters of the scene's
 * last wavefront sample pair — paths entering each depth, then shadow rays
 * per depth (2 x (max depth + 1) entries, n_out >= 18).  Synchronises. */
int mg_meshscene_queue_counts(mg_ctx* ctx, const mg_mesh_scene* s, int32_t n_out, uint32_t* out);
/* closest hit of n rays (device fp64 [n][6] = origin, direction): t (inf on
 * a miss) and the original triangle index (-1 on a miss); ties on t go to
 * the lower index (= a brute-force scan). */
int mg_meshscene_intersect(mg_ctx* ctx, const mg_mesh_scene* s, int32_t n, const double* rays,
                           double* t_out, int32_t* tri_out);
/* spp-sample render of the parameters theta (dtype [nobj][4][R*R]) into
 * img [3][H][W] (Philox iteration 0xffffffff, path = sample index). */
int mg_meshscene_render(mg_ctx* ctx, const mg_mesh_scene* s, int32_t dtype, int32_t W, int32_t H,
                        const double* view, int32_t spp, uint64_t key, const void* theta,
                        void* img);
/* One gradient sample pair over image rows [row0, row1): per pixel
 * prop_paths (n in [2, 8]) proportional paths j (path 0 = A, also evaluated
 * at theta_{t-1}) and one FD path C:
 *   prop = 2/(n(n-1)) sum_c sum_j (sum_{i != j} r_i) dI_j   (n = 2: r_A dI_B + r_B dI_A)
 *   diff = sum_c 2 r_C dI_A (theta_t) - 2 r_C dI_A (theta_{t-1})
 *   loss_out (device double) = 2/(n(n-1)) sum_c sum_{i<j} r_i r_j.
 * accum: device scratch of 2 * params int64 (internal layout), zero on
 * first use (left zeroed).  Exact fixed-point accumulation: tiles sum exactly to the full
 * pair.  prop = diff = NULL (wavefront form): the pair is left in accum as
 * the texel-interleaved fixed-point words [objects * R^2][prop | diff][nch]
 * for mg_meta_update_fixed to consume (which zeroes it) — no planar pair.  The scene owns the path-state workspace: calls on one scene must
 * be ordered (one stream at a time). */
int mg_meshscene_sample_pair(mg_ctx* ctx, mg_mesh_scene* s, int32_t dtype, int32_t W,
                             int32_t H, const double* view, const void* target_img,
                             const void* now, const void* prev, uint64_t key, uint32_t iteration,
                             int32_t row0, int32_t row1, int32_t prop_paths, void* accum,
                             void* prop, void* diff, double* loss_out);

/* Tile-sharded sample pair with the reduce-scatter fused into the adjoint
 * scatter: parameter j's contributions are added (2^-40 fixed-point int64
 * atomics, order independent) into rank (j / shard)'s accumulator
 * acc_ptrs[rank] = device int64 [2][shard] (prop | diff), typically peer
 * pointers of symmetric memory over NVLink.  world * shard must equal the
 * parameter count.  After all ranks' launches complete (a barrier), each
 * rank converts its own shard with mg_fixed_finalize. */
int mg_meshscene_sample_pair_sharded(mg_ctx* ctx, mg_mesh_scene* s, int32_t dtype, int32_t W,
                                     int32_t H, const double* view, const void* target_img,
                                     const void* now, const void* prev, uint64_t key,
                                     uint32_t iteration, int32_t row0, int32_t row1,
                                     int32_t prop_paths, int32_t world, void* const* acc_ptrs,
                                     int64_t shard, double* loss_out);
/* accum (device int64 [2][n], prop | diff in 2^-40 units) -> prop, diff
 * (dtype [n]); accum left zeroed. */
int mg_fixed_finalize(mg_ctx* ctx, int32_t dtype, int64_t n, void* accum, void* prop, void* diff);

/* ------------------------------- device-resident run_single (A13, A14) */
/* Per-replicate record of one coordinate plus scalars (harness.hpp:73-90;
 * full vectors are O(iterations*N) and are not recorded on the device). */
typedef struct mg_run_record {
  int32_t iterations_run;
  int32_t status;      /* 0 completed, 1 converged, 2 diverged (harness.hpp:74) */
  int64_t draws_used;
  int64_t evals_used;
} mg_run_record;

/* Series recorded per replicate per iteration, [R][iterations] fp64 each,
 * for coordinate cfg->coord (harness.cpp:219-244 extractor set). */
typedef struct mg_run_series {
  double* param_err;   /* ||params - truth|| (harness.cpp:212-215) */
  double* loss;
  double* prop;
  double* diff;
  double* grad_est;    /* meta mean / Adam m_hat */
  double* est_var;     /* meta var / Adam v_hat */
  double* alpha;       /* meta only */
  double* delta;
  double* true_grad;
  double* step_sq_norm;
  double* param;       /* params[coord] */
} mg_run_series;

/* run_single for replicates [rep_begin, rep_begin + rep_count) of cfg, on the
 * device, all replicates batched (harness.cpp:90-200 per replicate, the
 * std::thread pool of harness.cpp:249-272 becomes the grid).  Host arrays:
 * records[rep_count]; every non-NULL series pointer is a HOST array of
 * rep_count*iterations doubles (entries past iterations_run are NaN).
 * Optional final_params: host fp64 [rep_count][dim]. */
int mg_run_replicates(mg_ctx* ctx, const mg_experiment_config* cfg, int32_t rep_begin,
                      int32_t rep_count, mg_run_record* records, const mg_run_series* series,
                      double* final_params);

/* mg_run_replicates that also returns every RunRecord vector
 * (harness.hpp:79-88, recorded at harness.cpp:170-179): full is a HOST fp64
 * array [rep_count][iterations][8][dim] holding, per iteration, params,
 * prop, diff, mean_est, var_est, alpha (NaN for Adam), delta, true_grad;
 * NaN past iterations_run.  Feeds write_replicate_csv (harness.cpp:344-365). */
int mg_run_replicates_full(mg_ctx* ctx, const mg_experiment_config* cfg, int32_t rep_begin,
                           int32_t rep_count, mg_run_record* records, const mg_run_series* series,
                           double* final_params, double* full);

/* ---------------------------------- across-replicate aggregation (F2) */
/* Per-iteration statistics across replicates (harness.cpp:274-302,
 * stats.hpp:44-68), on the device.  series: device fp64 [S][R][T] (entry
 * [s][r][i] read only while i < iterations_run[r]); iterations_run: device
 * int32 [R].  Outputs (device): stats [S][5][T] = mean, variance (n-1),
 * median, q25, q75 of the active replicates — sums in replicate order, so
 * bit-identical to the reference; NaN sorts last — and optionally active[T]
 * (number of replicates with iterations_run > i).  R <= 8192. */
int mg_aggregate_series(mg_ctx* ctx, int32_t S, int32_t R, int32_t T, const double* series,
                        const int32_t* iterations_run, double* stats, int32_t* active);

/* run_experiment's replicate run + aggregation without the series leaving
 * the device: records[rep_count] as mg_run_replicates; stats: HOST fp64
 * [11][5][iterations] in mg_run_series field order; active: HOST int32
 * [iterations] or NULL. */
int mg_run_experiment_stats(mg_ctx* ctx, const mg_experiment_config* cfg, int32_t rep_begin,
                            int32_t rep_count, mg_run_record* records, double* stats,
                            int32_t* active);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* MGCUDA_H_ */
