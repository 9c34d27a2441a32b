// Drop-in replacement for the reference's metagrad/moment2.hpp
// (proj/include/metagrad/moment2.hpp:21-50): same class, constructors,
// accessors, exception types and messages; Moment2::step runs on the B200
// (mg_moment2_step, csrc/update.cu moment2_kernel).  Put
// include/metagrad_gpu ahead of the reference's include directory and the
// reference's harness and tests compile unchanged against it
// (tests/cpp/dropin/Makefile).
#pragma once

#include <cstdint>
#include <stdexcept>

#include "metagrad/vec.hpp"
#include "metagrad_gpu/backend.hpp"

namespace metagrad {

class Moment2 {
 public:
  explicit Moment2(double decay = 0.9) : s_{decay, 1.0, 0} {
    if (!(decay >= 0.0 && decay < 1.0))
      throw std::invalid_argument("Moment2: decay must lie in [0, 1)");
  }
  Moment2(double decay, Eigen::Index dim) : Moment2(decay) { m2_ = Vec::Zero(dim); }

  // moment2.hpp:30-39; decay^count is advanced by the ABI on the host by
  // repeated multiplication, exactly like the reference.
  void step(const Vec& x) {
    if (s_.count == 0 && m2_.size() == 0) m2_ = Vec::Zero(x.size());
    if (x.size() != m2_.size()) throw std::invalid_argument("Moment2: sample dimension mismatch");
    namespace g = metagrad_gpu;
    const g::Call c(x.size(), 2);  // slots: m2 (in/out), x
    c.put(0, m2_);
    c.put(1, x);
    c.upload(0, 2);
    g::check(mg_moment2_step(g::ctx(), MG_F64, x.size(), &s_, c.dev(0), c.dev(1)));
    c.download(0, 1);
    c.finish();
    c.get(0, m2_);
  }

  const Vec& m2() const { return m2_; }
  std::int64_t count() const { return s_.count; }
  double decay() const { return s_.decay; }

 private:
  mg_moment2_scalars s_;  // decay, decay^count, count
  Vec m2_;
};

}  // namespace metagrad
