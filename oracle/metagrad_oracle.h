/*
 * metagrad_oracle.h — CPU restatement of the reference hot path (fp64).
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  It is pinned against golden vectors produced by the UNMODIFIED
 * reference (oracle/_ref, built by oracle/ref/Makefile; fixtures in
 * tests/golden/, generator oracle/gen_golden.py).
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj).  Compiled with -ffp-contract=off so each a*b+c is
 * two roundings, as in the reference's Release build.
 */
#ifndef METAGRAD_ORACLE_H_
#define METAGRAD_ORACLE_H_

#include <stdint.h>

#include "../include/mgcuda.h" /* mg_experiment_config layout only */

#ifdef __cplusplus
extern "C" {
#endif

/* std::mt19937_64 (rng.hpp:36; libstdc++ random.h:1620-1627, random.tcc:328-470) */
typedef struct mgo_mt64 {
  uint64_t mt[312];
  int idx;
} mgo_mt64;

uint64_t mgo_mix64(uint64_t x);
void mgo_mt64_seed(mgo_mt64* g, uint64_t seed);
uint64_t mgo_mt64_next(mgo_mt64* g);
void mgo_rng_stream(mgo_mt64* g, uint64_t base_seed, uint64_t replicate);
double mgo_uniform(mgo_mt64* g);
double mgo_uniform_pos(mgo_mt64* g);
/* same modes as ref_rng_draws (oracle/ref/ref_capi.cpp) */
void mgo_rng_draws(uint64_t seed, uint64_t rep, int mode, int64_t n, void* out);

/* GF(2) jump-ahead of a block-boundary engine by g(A) (poly: 312 words) */
void mgo_mt64_jump(mgo_mt64* g, const uint64_t* poly, int deg);

/* Philox4x32-10 and the samplers' uniform mapping (scale mode, not in the
 * reference; see paper_2309_15676_b200/csrc/philox.cuh) */
void mgo_philox4x32_10(const uint32_t ctr[4], uint64_t key, uint32_t out[4]);
double mgo_philox_uniform(uint64_t key, uint32_t j, uint32_t it, uint32_t s, uint32_t st);

/* Moment2 (moment2.hpp:21-50) */
void mgo_moment2_step(int64_t n, double decay, double* decay_pow, int64_t* count, double* m2,
                      const double* x);

/* MetaEstimator::step (meta.hpp:90-113); returns 0, 1 (invalid_argument) or
 * 2 (logic_error). first_call performs the lazy init (:92-96). */
int mgo_meta_step(int64_t n, double lr, double eps_step, double eps_alpha, int clip, int first_call,
                  double* mean, double* var, double* alpha_prev, const double* prop,
                  const double* diff, const double* var_prop, const double* var_diff,
                  double* delta);

/* Adam::step (adam.hpp:23-37); s->beta*_pow and t advanced. */
void mgo_adam_step(int64_t n, mg_adam_scalars* s, double* m, double* v, const double* grad,
                   double* delta);

/* One fused meta-estimator iteration, the same computation as
 * mg_meta_update (include/mgcuda.h) in fp64 sequential order:
 * harness.cpp:144,153-157,160,182-188 + problems.cpp:214,225,228.
 * vprop/vdiff/target/prev may be NULL.  Returns 0 or an mg_status. */
int mgo_meta_update(int64_t n, const mg_meta_update_args* a, const double* prop, const double* diff,
                    const double* vprop, const double* vdiff, double* m2_prop, double* m2_diff,
                    double* mean, double* var, double* alpha_prev, const double* params_in,
                    double* params_out, const double* params_prev, const double* target,
                    mg_update_scalars* sc, double* delta_out);

/* Fused Adam iteration (mg_adam_update). */
void mgo_adam_update(int64_t n, mg_adam_scalars* s, int project, double proj_lo, const double* grad,
                     double* m, double* v, const double* params_in, double* params_out,
                     const double* target, mg_update_scalars* sc);

/* MiniRenderProblem (problems.cpp:162-228) */
void mgo_minirender_generate(int32_t pixel_count, uint64_t gen_seed, double exponent_max,
                             double* exponents, double* target);
void mgo_minirender_kernel_terms(int32_t pixel_count, int32_t spp, const double* exponents,
                                 const double* uniforms, double* cross, double* mean_basis);
/* draws P*spp uniforms from g; returns step_sq_norm */
double mgo_minirender_sample_pair(int32_t pixel_count, int32_t spp, const double* exponents,
                                  const double* target, mgo_mt64* g, const double* now,
                                  const double* prev, double* prop, double* diff);

/* ExpRateProblem (problems.cpp:30-94) */
double mgo_exprate_gradient_from_batch(double target_mean, int32_t n, double rate, double sum_c,
                                       double sum_c_sq);
/* returns 0 or MG_EDOMAIN */
int mgo_exprate_sample_pair(double target_mean, int32_t samples_per_iter, mgo_mt64* g,
                            double rate_now, double rate_prev, double* prop, double* diff,
                            double* ssn);

/* MultNoiseQuadratic (problems.cpp:99-157) */
double mgo_multnoise_sample_pair(int32_t dim, double sigma, int32_t samples_per_iter,
                                 const double* target, mgo_mt64* g, const double* now,
                                 const double* prev, double* prop, double* diff);

/* run_single (harness.cpp:90-200) with full per-iteration vectors.
 * Any output may be NULL; vector outputs are [iterations][dim].
 * Returns 0 or an mg_status (config errors).  rec gets status/counters. */
typedef struct mgo_full_record {
  double* params;
  double* loss;
  double* prop;
  double* diff;
  double* ssn;
  double* mean_est;
  double* var_est;
  double* alpha;
  double* delta;
  double* true_grad;
} mgo_full_record;

/* F1 slice: textured quad + rectangular area light, direct lighting (own
 * renderer).  tex/now/prev/prop/diff: [3][R*R]; images [3][H*W]. */
void mgo_quad_render(int W, int H, int R, const double* tex, const double Le[3], int spp,
                     uint64_t key, uint32_t st, double* img);
void mgo_quad_sample_pair(int W, int H, int R, const double Le[3], const double* target_img,
                          const double* now, const double* prev, uint64_t key, uint32_t it,
                          uint32_t st, double* prop, double* diff, double* loss_est);

/* F1 slice 2: helix of spheres, multi-bounce NEE, principled BSDF with 5
 * global parameters (base RGB, metal, rough) (own renderer).
 * sph: [nsph][4] (center, radius); images [3][H*W]. */
void mgo_helix_render(int W, int H, int nsph, const double* sph, const double Le[3],
                      const double env[3], const double ground[3], const double th[5], int spp,
                      uint64_t key, double* img);
void mgo_helix_sample_pair(int W, int H, int nsph, const double* sph, const double Le[3],
                           const double env[3], const double ground[3], const double* target_img,
                           const double now[5], const double prev[5], uint64_t key, uint32_t it,
                           double prop[5], double diff[5], double* loss_est);

int mgo_problem_dim(const mg_experiment_config* cfg);
int mgo_run_single(const mg_experiment_config* cfg, int32_t replicate, mg_run_record* rec,
                   const mgo_full_record* out);
/* run_single reduced to the device runner's coordinate series (mg_run_series). */
int mgo_run_single_series(const mg_experiment_config* cfg, int32_t replicate, mg_run_record* rec,
                          const mg_run_series* series, int32_t stride, double* final_params);

#ifdef __cplusplus
}
#endif

#endif

/* F1 slice 3: textured triangle-mesh scene (configs[3]); brute-force
 * intersection; triangle records [T][18] = v0 e1 e2 n uv0 duv1 duv2;
 * view[25] = cam fwd right up tan_half_fov light_y x0 x1 z0 z1 Le[3] env[3]
 * max_vertices; parameters [nobj][4][R*R] (base r,g,b, roughness). */
int mgo_mesh_closest_hit(int T, const double* tri, const double o[3], const double d[3],
                         double* t_out, double* u_out, double* v_out);
void mgo_mesh_render(int W, int H, int T, const double* tri, const int32_t* obj, int R,
                     const double* view, const double* theta, int spp, uint64_t key, double* img);
void mgo_mesh_sample_pair(int W, int H, int T, const double* tri, const int32_t* obj, int nobj,
                          int R, const double* view, const double* target_img, const double* now,
                          const double* prev, uint64_t key, uint32_t it, int row0, int row1,
                          double* prop, double* diff, double* loss_est);
int mgo_mesh_path_radiance(int W, int H, int T, const double* tri, const int32_t* obj, int R,
                           const double* view, const double* theta, int px, int py, uint64_t key,
                           uint32_t it, uint32_t path, double L_out[3]);
/* general form (configs[4]): nch = 4 (base rgb, rough; metal 0) or 5 (+ metal
 * as channel 4, full principled BSDF derivatives); nprop proportional paths
 * (2..8) plus the FD path. */
void mgo_meshx_render(int W, int H, int T, const double* tri, const int32_t* obj, int nch, int R,
                      const double* view, const double* theta, int spp, uint64_t key, double* img);
void mgo_meshx_sample_pair(int W, int H, int T, const double* tri, const int32_t* obj, int nobj,
                           int nch, int R, const double* view, const double* target_img,
                           const double* now, const double* prev, uint64_t key, uint32_t it,
                           int row0, int row1, int nprop, double* prop, double* diff,
                           double* loss_est);
int mgo_meshx_path_radiance(int W, int H, int T, const double* tri, const int32_t* obj, int nch,
                            int R, const double* view, const double* theta, int px, int py,
                            uint64_t key, uint32_t it, uint32_t path, double L_out[3]);
