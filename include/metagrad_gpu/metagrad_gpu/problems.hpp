// B200-backed gradient samplers behind the reference's Problem interface
// (proj/include/metagrad/problems.hpp:31-72): subclasses of
// the reference's MiniRenderProblem, ExpRateProblem and MultNoiseQuadratic
// whose sample_pair runs on the device (mg_minirender_sample_pair,
// mg_exprate_sample_pair, mg_multnoise_sample_pair) and otherwise inherit
// the reference's construction, true_gradient, loss, project and
// validate_params.  Use them wherever a metagrad::Problem is expected.
//
// The caller's Rng keeps its meaning: its std::mt19937_64 state (the only
// member of metagrad::Rng, rng.hpp:36 — standard-layout, so the two are
// pointer-interconvertible) is handed to a device engine before the draws
// and taken back after them, so the host stream continues exactly where
// the reference's own sample_pair would have left it.
#pragma once

#include <cstdint>
#include <random>
#include <sstream>
#include <string>
#include <type_traits>

#include "metagrad/problems.hpp"
#include "metagrad_gpu/backend.hpp"

namespace metagrad_gpu {

inline std::mt19937_64& engine_of(metagrad::Rng& rng) {
  static_assert(std::is_standard_layout<metagrad::Rng>::value &&
                    sizeof(metagrad::Rng) == sizeof(std::mt19937_64),
                "metagrad::Rng is expected to hold exactly one std::mt19937_64");
  return *reinterpret_cast<std::mt19937_64*>(&rng);
}

// For one sample_pair call: the host engine's state moves into this
// thread's device engine; finish() moves the advanced state back.
class EngineLease {
 public:
  explicit EngineLease(metagrad::Rng& rng) : host_(engine_of(rng)), t_(thread_state()) {
    if (!t_.engine) {
      const std::uint64_t seed = 5489u;
      check(mg_mt64_create(t_.ctx, 1, &seed, &t_.engine));
    }
    // libstdc++ serialises the engine as its 312 state words and position
    std::stringstream ss;
    ss << host_;
    std::uint64_t words[312];
    for (auto& w : words) ss >> w;
    std::int32_t idx = 0;
    ss >> idx;
    check(mg_mt64_set_state(t_.ctx, t_.engine, 0, words, idx));
  }
  mg_mt64* get() const { return t_.engine; }
  void finish() const {
    std::uint64_t words[312];
    std::int32_t idx = 0;
    check(mg_mt64_get_state(t_.ctx, t_.engine, 0, words, &idx));
    std::stringstream ss;
    for (auto w : words) ss << w << ' ';
    ss << idx;
    ss >> host_;
  }

 private:
  std::mt19937_64& host_;
  ThreadState& t_;
};

class MiniRenderProblem : public metagrad::MiniRenderProblem {
 public:
  using metagrad::MiniRenderProblem::MiniRenderProblem;

  metagrad::GradientSamplePair sample_pair(const metagrad::Vec& now, const metagrad::Vec& prev,
                                           metagrad::Rng& rng) const override {
    validate_params(now);
    validate_params(prev);
    const Eigen::Index P = dim();
    // [0] exponents [1] target [2] now [3] prev | [4] prop [5] diff [6] ssn
    const Call call(P, 7);
    call.put(0, shape_exponents());
    call.put(1, target_image());
    call.put(2, now);
    call.put(3, prev);
    call.upload(0, 4);
    const EngineLease eng(rng);
    check(mg_minirender_sample_pair(ctx(), MG_F64, 1, int32_t(P), spp(), call.dev(0), call.dev(1),
                                    eng.get(), call.dev(2), call.dev(3), call.dev(4),
                                    call.dev(5), call.dev(6)));
    call.download(4, 3);
    call.finish();
    eng.finish();
    metagrad::GradientSamplePair pair;
    call.get(4, pair.prop);
    call.get(5, pair.diff);
    pair.step_sq_norm = call.host(6)[0];
    return pair;
  }
};

class ExpRateProblem : public metagrad::ExpRateProblem {
 public:
  using metagrad::ExpRateProblem::ExpRateProblem;

  metagrad::GradientSamplePair sample_pair(const metagrad::Vec& now, const metagrad::Vec& prev,
                                           metagrad::Rng& rng) const override {
    validate_params(now);
    validate_params(prev);
    // [0] rate_now [1] rate_prev | [2] prop [3] diff [4] ssn
    const Call call(1, 5);
    call.put(0, now);
    call.put(1, prev);
    call.upload(0, 2);
    const EngineLease eng(rng);
    check(mg_exprate_sample_pair(ctx(), 1, target_mean(), samples_per_iter(), eng.get(),
                                 call.dev(0), call.dev(1), call.dev(2), call.dev(3), call.dev(4)));
    call.download(2, 3);
    call.finish();
    eng.finish();
    metagrad::GradientSamplePair pair;
    call.get(2, pair.prop);
    call.get(3, pair.diff);
    pair.step_sq_norm = call.host(4)[0];
    return pair;
  }
};

class MultNoiseQuadratic : public metagrad::MultNoiseQuadratic {
 public:
  using metagrad::MultNoiseQuadratic::MultNoiseQuadratic;

  metagrad::GradientSamplePair sample_pair(const metagrad::Vec& now, const metagrad::Vec& prev,
                                           metagrad::Rng& rng) const override {
    validate_params(now);
    validate_params(prev);
    const Eigen::Index d = dim();
    // [0] target [1] now [2] prev | [3] prop [4] diff [5] ssn
    const Call call(d, 6);
    call.put(0, *truth_params());
    call.put(1, now);
    call.put(2, prev);
    call.upload(0, 3);
    const EngineLease eng(rng);
    check(mg_multnoise_sample_pair(ctx(), 1, int32_t(d), noise_amp(), samples_per_iter(),
                                   call.dev(0), eng.get(), call.dev(1), call.dev(2), call.dev(3),
                                   call.dev(4), call.dev(5)));
    call.download(3, 3);
    call.finish();
    eng.finish();
    metagrad::GradientSamplePair pair;
    call.get(3, pair.prop);
    call.get(4, pair.diff);
    pair.step_sq_norm = call.host(5)[0];
    return pair;
  }
};

}  // namespace metagrad_gpu
