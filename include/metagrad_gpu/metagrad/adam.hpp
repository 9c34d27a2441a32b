// Drop-in for the reference header metagrad/adam.hpp
// (proj/include/metagrad/adam.hpp:14-50): class Adam with the same
// constructor defaults, accessors, exceptions and messages; the update and
// the bias corrections run on the B200 (mg_adam_step, mg_scalar_op).
// beta^t advances on the host by repeated multiplication inside the ABI,
// as in the reference.
#pragma once

#include "metagrad_gpu/backend.hpp"

namespace metagrad {

class Adam {
  mg_adam_scalars s_;  // {lr, beta1, beta2, eps, beta1^t, beta2^t, t}
  Vec m_, v_;

  static Vec bias_corrected(const Vec& x, double one_minus_pow) {
    namespace g = metagrad_gpu;
    const g::Call call(x.size(), 2);  // [0] moment, [1] corrected
    call.put(0, x);
    call.upload(0, 1);
    g::check(mg_scalar_op(g::ctx(), MG_F64, x.size(), call.dev(0), one_minus_pow, 1, call.dev(1)));
    call.download(1, 1);
    call.finish();
    return call.get(1);
  }

 public:
  explicit Adam(double lr, double beta1 = 0.9, double beta2 = 0.999, double eps = 1e-8)
      : s_{lr, beta1, beta2, eps, 1.0, 1.0, 0} {
    metagrad_gpu::require(lr > 0.0, "Adam: lr must be positive");
    const bool b1 = beta1 >= 0.0 && beta1 < 1.0, b2 = beta2 >= 0.0 && beta2 < 1.0;
    metagrad_gpu::require(b1 && b2, "Adam: betas must lie in [0, 1)");
  }

  std::int64_t t() const { return s_.t; }
  const Vec& m() const { return m_; }
  const Vec& v() const { return v_; }
  Vec m_hat() const { return s_.t == 0 ? m_ : bias_corrected(m_, 1.0 - s_.beta1_pow); }
  Vec v_hat() const { return s_.t == 0 ? v_ : bias_corrected(v_, 1.0 - s_.beta2_pow); }

  // adam.hpp:23-37
  Vec step(const Vec& g_in) {
    namespace g = metagrad_gpu;
    const Eigen::Index n = g_in.size();
    if (m_.size() == 0 && s_.t == 0) m_ = v_ = Vec::Zero(n);
    g::require(m_.size() == n, "Adam: gradient dimension mismatch");
    const g::Call call(n, 4);  // [0] m, [1] v in/out, [2] gradient, [3] step
    call.put(0, m_);
    call.put(1, v_);
    call.put(2, g_in);
    call.upload(0, 3);
    g::check(mg_adam_step(g::ctx(), MG_F64, n, &s_, call.dev(0), call.dev(1), call.dev(2),
                          call.dev(3)));
    call.download(0, 2);
    call.download(3, 1);
    call.finish();
    call.get(0, m_);
    call.get(1, v_);
    return call.get(3);
  }
};

}  // namespace metagrad
