// Drop-in for the reference header metagrad/moment2.hpp
// (proj/include/metagrad/moment2.hpp:21-50): class Moment2 with the same
// constructors, accessors, exceptions and messages; step() runs on the B200
// (mg_moment2_step -> csrc/update.cu moment2_kernel).  Search
// include/metagrad_gpu before the reference's include directory and the
// reference's harness and tests compile unchanged against it
// (tests/cpp/dropin/Makefile).
#pragma once

#include "metagrad_gpu/backend.hpp"

namespace metagrad {

class Moment2 {
  mg_moment2_scalars s_;  // {decay, decay^count, count}; advanced by the ABI on the host
  Vec m2_;

 public:
  explicit Moment2(double decay = 0.9) : s_{decay, 1.0, 0} {
    metagrad_gpu::require(decay >= 0.0 && decay < 1.0, "Moment2: decay must lie in [0, 1)");
  }
  Moment2(double decay, Eigen::Index dim) : Moment2(decay) { m2_ = Vec::Zero(dim); }

  double decay() const { return s_.decay; }
  std::int64_t count() const { return s_.count; }
  const Vec& m2() const { return m2_; }

  // moment2.hpp:30-39 — lazily sized on the first sample
  void step(const Vec& x) {
    namespace g = metagrad_gpu;
    if (m2_.size() == 0 && s_.count == 0) m2_ = Vec::Zero(x.size());
    g::require(m2_.size() == x.size(), "Moment2: sample dimension mismatch");
    const g::Call call(x.size(), 2);  // [0] m2 in/out, [1] sample
    call.put(0, m2_);
    call.put(1, x);
    call.upload(0, 2);
    g::check(mg_moment2_step(g::ctx(), MG_F64, x.size(), &s_, call.dev(0), call.dev(1)));
    call.download(0, 1);
    call.finish();
    call.get(0, m2_);
  }
};

}  // namespace metagrad
