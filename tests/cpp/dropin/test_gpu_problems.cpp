// B200 samplers behind the reference's Problem interface
// (include/metagrad_gpu/metagrad_gpu/problems.hpp) against the reference's
// own CPU samplers (proj/src/problems.cpp, compiled into libmetagrad_gpu.so):
// same draws from the same Rng, same pairs (bit-exact for mult-noise, pow /
// log tolerance for mini-render / exp-rate as in DESIGN.md §5), the caller's
// Rng left at exactly the same position, the same exceptions, and a
// reference-style optimisation loop (harness.cpp:90-200 shape) over the
// drop-in estimators.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cmath>
#include <cstring>
#include <stdexcept>

#include "metagrad/meta.hpp"
#include "metagrad/moment2.hpp"
#include "metagrad/problems.hpp"
#include "metagrad/rng.hpp"
#include "metagrad_gpu/problems.hpp"

using metagrad::GradientSamplePair;
using metagrad::Rng;
using metagrad::Vec;

namespace {

double max_rel(const Vec& a, const Vec& b, double floor) {
  double m = 0.0;
  for (Eigen::Index j = 0; j < a.size(); ++j) {
    const double s = std::max({std::fabs(a[j]), std::fabs(b[j]), floor});
    m = std::max(m, std::fabs(a[j] - b[j]) / s);
  }
  return m;
}

bool same_bits(const Vec& a, const Vec& b) {
  if (a.size() != b.size()) return false;
  for (Eigen::Index j = 0; j < a.size(); ++j) {
    const double x = a[j], y = b[j];
    if (std::memcmp(&x, &y, sizeof(double)) != 0) return false;
  }
  return true;
}

// Both problems over `iters` pairs on twin Rngs; returns the worst relative
// difference of prop/diff and checks the Rngs stay in lockstep.
template <class Ref, class Gpu>
double compare(const Ref& ref, const Gpu& gpu, Vec params, int iters, std::uint64_t seed,
               bool exact) {
  Rng r1 = Rng::stream(seed, 3), r2 = Rng::stream(seed, 3);
  Vec prev = params;
  double worst = 0.0;
  for (int i = 0; i < iters; ++i) {
    const GradientSamplePair a = ref.sample_pair(params, prev, r1);
    const GradientSamplePair b = gpu.sample_pair(params, prev, r2);
    if (exact) {
      CHECK(same_bits(a.prop, b.prop));
      CHECK(same_bits(a.diff, b.diff));
      CHECK(a.step_sq_norm == b.step_sq_norm);
    } else {
      worst = std::max(worst, max_rel(a.prop, b.prop, 1e-3));
      worst = std::max(worst, max_rel(a.diff, b.diff, 1e-6));
      CHECK(std::fabs(a.step_sq_norm - b.step_sq_norm) <= 1e-12 * (1.0 + a.step_sq_norm));
    }
    if (i == 0) CHECK(b.step_sq_norm == 0.0);
    Rng c1 = r1, c2 = r2;  // host streams continue identically
    CHECK(c1.raw() == c2.raw());
    prev = params;
    params = params * 0.97 + 0.01;
  }
  return worst;
}

}  // namespace

TEST_CASE("gpu mult-noise sample_pair is bit-identical and keeps the Rng in step") {
  Vec target = Vec::Zero(5);
  target << 0.5, -1.0, 2.0, 0.0, 3.0;
  const metagrad::MultNoiseQuadratic ref(target, 0.7, 3);
  const metagrad_gpu::MultNoiseQuadratic gpu(target, 0.7, 3);
  compare(ref, gpu, Vec::Constant(5, 2.0), 12, 42, true);
}

TEST_CASE("gpu mini-render sample_pair matches the reference (pow tolerance)") {
  const metagrad::MiniRenderProblem ref(300, 4, 2024);
  const metagrad_gpu::MiniRenderProblem gpu(300, 4, 2024);
  const double worst = compare(ref, gpu, Vec::Constant(300, 0.3), 8, 7, false);
  CAPTURE(worst);
  CHECK(worst < 1e-9);
}

TEST_CASE("gpu exp-rate sample_pair matches the reference (log tolerance)") {
  const metagrad::ExpRateProblem ref(2.0, 32, 2.0);
  const metagrad_gpu::ExpRateProblem gpu(2.0, 32, 2.0);
  const double worst = compare(ref, gpu, Vec::Constant(1, 1.3), 20, 11, false);
  CAPTURE(worst);
  CHECK(worst < 1e-11);
}

TEST_CASE("gpu exp-rate rejects non-positive rates without consuming draws") {
  const metagrad_gpu::ExpRateProblem gpu(2.0, 8, 2.0);
  Rng r1(99), r2(99);
  CHECK_THROWS_AS(gpu.sample_pair(Vec::Constant(1, -1.0), Vec::Constant(1, 1.0), r1),
                  std::domain_error);
  CHECK(r1.raw() == r2.raw());
}

TEST_CASE("variance_empirical runs through the gpu sampler") {
  Vec target = Vec::Zero(2);
  target << 1.0, -1.0;
  const metagrad::MultNoiseQuadratic ref(target, 0.5, 2);
  const metagrad_gpu::MultNoiseQuadratic gpu(target, 0.5, 2);
  Rng r1(5), r2(5);
  const Vec now = Vec::Constant(2, 0.5), prev = Vec::Constant(2, 0.45);
  const auto a = ref.variance_empirical(now, prev, 50, r1);
  const auto b = gpu.variance_empirical(now, prev, 50, r2);
  CHECK(same_bits(a.prop, b.prop));
  CHECK(same_bits(a.diff, b.diff));
}

TEST_CASE("reference-style meta loop over gpu sampler and gpu estimators converges") {
  // harness.cpp:108-188 in miniature: Moment2 x2 (drop-in), global-norm
  // decoupling, MetaEstimator (drop-in), update, projection.
  const metagrad_gpu::MiniRenderProblem prob(64, 4, 1234);
  Rng rng = Rng::stream(0, 0);
  Vec params = prob.initial_params(), prev = params;
  metagrad::Moment2 mp(0.9), md(0.5);
  metagrad::MetaEstimator meta(0.02);
  const double err0 = std::sqrt((params - *prob.truth_params()).square().sum());
  for (int i = 0; i < 300; ++i) {
    const GradientSamplePair pair = prob.sample_pair(params, prev, rng);
    mp.step(pair.prop);
    if (pair.step_sq_norm > 0.0) md.step(pair.diff / std::sqrt(pair.step_sq_norm));
    const Vec var_diff = md.count() > 0 ? metagrad::rescale_diff_variance(md.m2(), pair.step_sq_norm)
                                        : Vec(Vec::Zero(params.size()));
    const Vec delta = meta.step(pair, mp.m2(), var_diff);
    prev = params;
    params = params + delta;
    prob.project(params);
  }
  const double err1 = std::sqrt((params - *prob.truth_params()).square().sum());
  CAPTURE(err0);
  CAPTURE(err1);
  CHECK(err1 < 0.5 * err0);
}
