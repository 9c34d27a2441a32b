// Drop-in for the reference header metagrad/meta.hpp
// (proj/include/metagrad/meta.hpp:1-116): GradientSamplePair, clip_alpha,
// compute_alpha, rescale_diff_variance and MetaEstimator with the same
// public members, defaults, exceptions and messages.  Vector arithmetic
// runs on the B200 (mg_meta_step, mg_compute_alpha, mg_scalar_op);
// clip_alpha is the reference's scalar helper, restated.
#pragma once

#include <algorithm>
#include <limits>

#include "metagrad_gpu/backend.hpp"

namespace metagrad {

constexpr double kDefaultEpsStep = 1e-8, kDefaultEpsAlpha = 1e-30;

// meta.hpp:20-24 — one iteration's proportional and finite-difference samples
struct GradientSamplePair { Vec prop, diff; double step_sq_norm = 0.0; };

// meta.hpp:30-32: the weight bound 1 / (2 - alpha_prev)
inline double clip_alpha(double raw, double alpha_prev) {
  const double bound = 1.0 / (2.0 - alpha_prev);
  return std::min(raw, bound);
}

// meta.hpp:38-47
inline Vec compute_alpha(const Vec& var_prop, const Vec& var_meta, const Vec& var_diff,
                         const Vec& alpha_prev, double eps_alpha = kDefaultEpsAlpha) {
  namespace g = metagrad_gpu;
  const Eigen::Index n = var_prop.size();
  g::require(var_meta.size() == n && var_diff.size() == n && alpha_prev.size() == n,
             "compute_alpha: dimension mismatch");
  const g::Call call(n, 5);  // [0..3] inputs, [4] weights
  call.put(0, var_prop);
  call.put(1, var_meta);
  call.put(2, var_diff);
  call.put(3, alpha_prev);
  call.upload(0, 4);
  g::check(mg_compute_alpha(g::ctx(), MG_F64, n, call.dev(0), call.dev(1), call.dev(2),
                            call.dev(3), eps_alpha, call.dev(4)));
  call.download(4, 1);
  call.finish();
  return call.get(4);
}

// meta.hpp:51-53: Var[diff] = Var[diff / ||step||] * ||step||^2
inline Vec rescale_diff_variance(const Vec& var_diff_decoupled, double step_sq_norm) {
  namespace g = metagrad_gpu;
  const g::Call call(var_diff_decoupled.size(), 2);
  call.put(0, var_diff_decoupled);
  call.upload(0, 1);
  g::check(mg_scalar_op(g::ctx(), MG_F64, var_diff_decoupled.size(), call.dev(0), step_sq_norm,
                        0, call.dev(1)));
  call.download(1, 1);
  call.finish();
  return call.get(1);
}

// meta.hpp:71-114 — public state so callers (and the reference's tests) can
// inject it; the device sees it only for the duration of step().
struct MetaEstimator {
  double lr = 0.001, eps_step = kDefaultEpsStep, eps_alpha = kDefaultEpsAlpha;
  bool clip_enabled = true;
  Vec mean, var, alpha_prev;

  explicit MetaEstimator(double lr_ = 0.001, double eps_step_ = kDefaultEpsStep,
                         double eps_alpha_ = kDefaultEpsAlpha)
      : lr(lr_), eps_step(eps_step_), eps_alpha(eps_alpha_) {
    metagrad_gpu::require(lr > 0.0, "MetaEstimator: lr must be positive");
  }

  Vec step(const GradientSamplePair& sample, const Vec& var_prop, const Vec& var_diff) {
    namespace g = metagrad_gpu;
    const Eigen::Index n = sample.prop.size();
    if (mean.size() == 0) {  // lazy initialisation, meta.hpp:92-96
      mean = var = Vec::Zero(n);
      alpha_prev = Vec::Constant(n, -std::numeric_limits<double>::infinity());
    }
    const bool sizes_ok = sample.diff.size() == n && var_prop.size() == n &&
                          var_diff.size() == n && mean.size() == n && var.size() == n &&
                          alpha_prev.size() == n;
    g::require(sizes_ok, "MetaEstimator: dimension mismatch");
    // [0] mean [1] var [2] alpha_prev (in/out), [3] prop [4] diff [5] var_prop
    // [6] var_diff, [7] parameter step
    const g::Call call(n, 8);
    const Vec* in[7] = {&mean, &var, &alpha_prev, &sample.prop, &sample.diff, &var_prop, &var_diff};
    for (int k = 0; k < 7; ++k) call.put(k, *in[k]);
    call.upload(0, 7);
    const mg_meta_params hp{lr, eps_step, eps_alpha, clip_enabled ? 1 : 0};
    // the negative-variance check (meta.hpp:100-101) precedes any state
    // change; the host state is replaced only on success
    g::check(mg_meta_step(g::ctx(), MG_F64, n, &hp, 0, call.dev(0), call.dev(1), call.dev(2),
                          call.dev(3), call.dev(4), call.dev(5), call.dev(6), call.dev(7)));
    call.download(0, 3);
    call.download(7, 1);
    call.finish();
    call.get(0, mean);
    call.get(1, var);
    call.get(2, alpha_prev);
    return call.get(7);
  }
};

}  // namespace metagrad
