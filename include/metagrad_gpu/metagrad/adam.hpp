// Drop-in replacement for the reference's metagrad/adam.hpp
// (proj/include/metagrad/adam.hpp:14-50): same class, defaults, accessors,
// exception types and messages; the update and the bias corrections run on
// the B200 (mg_adam_step, mg_scalar_op).  beta^t is advanced by the ABI on
// the host by repeated multiplication, like the reference.
#pragma once

#include <cstdint>
#include <stdexcept>

#include "metagrad/vec.hpp"
#include "metagrad_gpu/backend.hpp"

namespace metagrad {

class Adam {
 public:
  explicit Adam(double lr, double beta1 = 0.9, double beta2 = 0.999, double eps = 1e-8)
      : s_{lr, beta1, beta2, eps, 1.0, 1.0, 0} {
    if (!(lr > 0.0)) throw std::invalid_argument("Adam: lr must be positive");
    if (!(beta1 >= 0.0 && beta1 < 1.0) || !(beta2 >= 0.0 && beta2 < 1.0))
      throw std::invalid_argument("Adam: betas must lie in [0, 1)");
  }

  Vec step(const Vec& grad) {
    if (s_.t == 0 && m_.size() == 0) {
      m_ = Vec::Zero(grad.size());
      v_ = Vec::Zero(grad.size());
    }
    if (grad.size() != m_.size()) throw std::invalid_argument("Adam: gradient dimension mismatch");
    namespace g = metagrad_gpu;
    const g::Call c(grad.size(), 4);  // slots: m, v (in/out), grad, delta
    c.put(0, m_);
    c.put(1, v_);
    c.put(2, grad);
    c.upload(0, 3);
    g::check(mg_adam_step(g::ctx(), MG_F64, grad.size(), &s_, c.dev(0), c.dev(1), c.dev(2),
                          c.dev(3)));
    c.download(0, 2);
    c.download(3, 1);
    c.finish();
    c.get(0, m_);
    c.get(1, v_);
    return c.get(3);
  }

  std::int64_t t() const { return s_.t; }
  const Vec& m() const { return m_; }
  const Vec& v() const { return v_; }
  Vec m_hat() const { return s_.t > 0 ? corrected(m_, 1.0 - s_.beta1_pow) : m_; }
  Vec v_hat() const { return s_.t > 0 ? corrected(v_, 1.0 - s_.beta2_pow) : v_; }

 private:
  static Vec corrected(const Vec& x, double denom) {
    namespace g = metagrad_gpu;
    const g::Call c(x.size(), 2);  // slots: x, out
    c.put(0, x);
    c.upload(0, 1);
    g::check(mg_scalar_op(g::ctx(), MG_F64, x.size(), c.dev(0), denom, 1, c.dev(1)));
    c.download(1, 1);
    c.finish();
    return c.get(1);
  }
  mg_adam_scalars s_;  // lr, beta1, beta2, eps, beta1^t, beta2^t, t
  Vec m_, v_;
};

}  // namespace metagrad
