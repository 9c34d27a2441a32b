// Drop-in replacement for the reference's metagrad/meta.hpp
// (proj/include/metagrad/meta.hpp:1-116): GradientSamplePair, clip_alpha,
// compute_alpha, rescale_diff_variance and MetaEstimator with the same
// public members, defaults, exception types and messages.  The vector
// arithmetic runs on the B200 (mg_meta_step, mg_compute_alpha,
// mg_scalar_op); clip_alpha is the reference's scalar helper.
#pragma once

#include <algorithm>
#include <limits>
#include <stdexcept>

#include "metagrad/vec.hpp"
#include "metagrad_gpu/backend.hpp"

namespace metagrad {

constexpr double kDefaultEpsAlpha = 1e-30;
constexpr double kDefaultEpsStep = 1e-8;

// meta.hpp:20-24
struct GradientSamplePair {
  Vec prop;
  Vec diff;
  double step_sq_norm = 0.0;
};

// meta.hpp:30-32 (scalar)
inline double clip_alpha(double raw, double alpha_prev) {
  return std::min(raw, 1.0 / (2.0 - alpha_prev));
}

// meta.hpp:38-47
inline Vec compute_alpha(const Vec& var_prop, const Vec& var_meta, const Vec& var_diff,
                         const Vec& alpha_prev, double eps_alpha = kDefaultEpsAlpha) {
  if (var_meta.size() != var_prop.size() || var_diff.size() != var_prop.size() ||
      alpha_prev.size() != var_prop.size())
    throw std::invalid_argument("compute_alpha: dimension mismatch");
  namespace g = metagrad_gpu;
  const g::Call c(var_prop.size(), 5);  // slots: vp, vm, vd, alpha_prev, out
  c.put(0, var_prop);
  c.put(1, var_meta);
  c.put(2, var_diff);
  c.put(3, alpha_prev);
  c.upload(0, 4);
  g::check(mg_compute_alpha(g::ctx(), MG_F64, var_prop.size(), c.dev(0), c.dev(1), c.dev(2),
                            c.dev(3), eps_alpha, c.dev(4)));
  c.download(4, 1);
  c.finish();
  return c.get(4);
}

// meta.hpp:51-53
inline Vec rescale_diff_variance(const Vec& var_diff_decoupled, double step_sq_norm) {
  namespace g = metagrad_gpu;
  const g::Call c(var_diff_decoupled.size(), 2);  // slots: x, out
  c.put(0, var_diff_decoupled);
  c.upload(0, 1);
  g::check(mg_scalar_op(g::ctx(), MG_F64, var_diff_decoupled.size(), c.dev(0), step_sq_norm, 0,
                        c.dev(1)));
  c.download(1, 1);
  c.finish();
  return c.get(1);
}

// meta.hpp:71-114
struct MetaEstimator {
  double lr = 0.001;
  double eps_step = kDefaultEpsStep;
  double eps_alpha = kDefaultEpsAlpha;
  bool clip_enabled = true;

  Vec mean;
  Vec var;
  Vec alpha_prev;

  explicit MetaEstimator(double lr_ = 0.001, double eps_step_ = kDefaultEpsStep,
                         double eps_alpha_ = kDefaultEpsAlpha)
      : lr(lr_), eps_step(eps_step_), eps_alpha(eps_alpha_) {
    if (!(lr > 0.0)) throw std::invalid_argument("MetaEstimator: lr must be positive");
  }

  Vec step(const GradientSamplePair& sample, const Vec& var_prop, const Vec& var_diff) {
    const Eigen::Index n = sample.prop.size();
    if (mean.size() == 0) {  // meta.hpp:92-96
      mean = Vec::Zero(n);
      var = Vec::Zero(n);
      alpha_prev = Vec::Constant(n, -std::numeric_limits<double>::infinity());
    }
    if (sample.diff.size() != n || var_prop.size() != n || var_diff.size() != n ||
        mean.size() != n || var.size() != n || alpha_prev.size() != n)
      throw std::invalid_argument("MetaEstimator: dimension mismatch");
    namespace g = metagrad_gpu;
    // slots: mean, var, alpha_prev (in/out), prop, diff, var_prop, var_diff, delta
    const g::Call c(n, 8);
    c.put(0, mean);
    c.put(1, var);
    c.put(2, alpha_prev);
    c.put(3, sample.prop);
    c.put(4, sample.diff);
    c.put(5, var_prop);
    c.put(6, var_diff);
    c.upload(0, 7);
    const mg_meta_params p{lr, eps_step, eps_alpha, clip_enabled ? 1 : 0};
    // the negative-variance check (meta.hpp:100-101) runs before any state
    // changes; the host state is only replaced on success
    g::check(mg_meta_step(g::ctx(), MG_F64, n, &p, 0, c.dev(0), c.dev(1), c.dev(2), c.dev(3),
                          c.dev(4), c.dev(5), c.dev(6), c.dev(7)));
    c.download(0, 3);
    c.download(7, 1);
    c.finish();
    c.get(0, mean);
    c.get(1, var);
    c.get(2, alpha_prev);
    return c.get(7);
  }
};

}  // namespace metagrad
