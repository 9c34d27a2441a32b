// The reference's own unit-test cases (proj/tests/test_moment2.cpp,
// test_meta.cpp, test_adam.cpp, test_problems.cpp), restated against the
// B200 C++ adapter (include/mgcuda.hpp): same expectations, same
// tolerances, device vectors instead of Eigen arrays.  Built by
// tests/cpp/Makefile, run by tests/test_gpu_cpp_adapter.py (-m gpu).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cmath>
#include <limits>
#include <random>
#include <vector>

#include "mgcuda.hpp"

using namespace mgcuda;
using V = std::vector<double>;

namespace {
Context& ctx() {
  static Context c(0);
  return c;
}
DeviceVec<double> dv(const V& v) { return DeviceVec<double>::from_host(ctx(), v); }
const double kNegInf = -std::numeric_limits<double>::infinity();
}  // namespace

// test_moment2.cpp:41-46
TEST_CASE("first step is the raw square") {
  Moment2<> ema(ctx(), 0.9);
  ema.step(dv({3.0}));
  CHECK(ema.count() == 1);
  CHECK(ema.m2().to_host()[0] == 9.0);
}

// test_moment2.cpp:48-58
TEST_CASE("two steps match the closed form") {
  Moment2<> ema(ctx(), 0.9);
  ema.step(dv({1.0}));
  ema.step(dv({2.0}));
  CHECK(ema.m2().to_host()[0] == doctest::Approx(0.49 / 0.19).epsilon(1e-12));
}

// test_moment2.cpp:35-39
TEST_CASE("degenerate decay is rejected") {
  CHECK_THROWS_AS(Moment2<>(ctx(), 1.0), std::invalid_argument);
  CHECK_THROWS_AS(Moment2<>(ctx(), -0.1), std::invalid_argument);
}

// test_moment2.cpp:119-123
TEST_CASE("dimension mismatch is rejected") {
  Moment2<> ema(ctx(), 0.9);
  ema.step(dv({0.0, 0.0, 0.0}));
  CHECK_THROWS_AS(ema.step(dv({0.0, 0.0})), std::invalid_argument);
}

// test_moment2.cpp:125-130
TEST_CASE("non-finite samples propagate") {
  Moment2<> ema(ctx(), 0.9);
  ema.step(dv({1.0}));
  ema.step(dv({std::nan("")}));
  CHECK(std::isnan(ema.m2().to_host()[0]));
}

// test_meta.cpp:153-157: raw weight below the bound passes through
TEST_CASE("meta: injected alpha_prev 0.5, var 1 -> alpha 0.5") {
  MetaEstimator<> meta(ctx(), 0.01);
  meta.mean = dv({0.0});
  meta.var = dv({1.0});
  meta.alpha_prev = dv({0.5});
  GradientSamplePair<> pair{dv({0.0}), dv({0.0}), 0.0};
  meta.step(pair, dv({1.0}), dv({0.0}));
  CHECK(meta.alpha_prev.to_host()[0] == doctest::Approx(0.5).epsilon(1e-14));
}

// test_meta.cpp:200-211
TEST_CASE("first meta step collapses to the proportional sample") {
  MetaEstimator<> meta(ctx(), 0.01);
  GradientSamplePair<> pair{dv({1.25, 1.25}), dv({0.0, 0.0}), 0.0};
  const auto delta = meta.step(pair, dv({0.64, 0.64}), dv({0.0, 0.0})).to_host();
  CHECK(meta.mean.to_host() == V({1.25, 1.25}));
  CHECK(meta.var.to_host() == V({0.64, 0.64}));
  for (double d : delta) CHECK(d == doctest::Approx(-0.01 * 1.25 / (0.8 + 1e-8)).epsilon(1e-14));
  CHECK(meta.alpha_prev.to_host()[0] == 0.0);  // -inf sentinel forces alpha = 0
}

// test_meta.cpp:213-226
TEST_CASE("hand-evaluated step from an injected state") {
  MetaEstimator<> meta(ctx(), 0.01);
  meta.mean = dv({0.0});
  meta.var = dv({1.0});
  meta.alpha_prev = dv({0.5});
  GradientSamplePair<> pair{dv({2.0}), dv({1.0}), 0.01};
  meta.step(pair, dv({1.0}), dv({0.0}));
  CHECK(meta.alpha_prev.to_host()[0] == doctest::Approx(0.5).epsilon(1e-14));
  CHECK(meta.mean.to_host()[0] == doctest::Approx(1.5).epsilon(1e-14));
  CHECK(meta.var.to_host()[0] == doctest::Approx(0.5).epsilon(1e-14));
}

// test_meta.cpp:228-244 (1000 steps here)
TEST_CASE("zero diffs and constant variance give the perfect running average") {
  const double v = 1.5;
  std::mt19937_64 gen(99);
  MetaEstimator<> meta(ctx(), 0.01);
  long double run_avg = 0.0L;
  for (int i = 0; i < 1000; ++i) {
    const double p = 0.5 + double(gen() >> 11) * 0x1.0p-53;
    GradientSamplePair<> pair{dv({p}), dv({0.0}), 0.0};
    meta.step(pair, dv({v}), dv({0.0}));
    run_avg += (static_cast<long double>(p) - run_avg) / (i + 1);
    if (i % 97 == 0 || i == 999) {
      const double var_expected = v / double(i + 1);
      CHECK(std::abs(meta.var.to_host()[0] - var_expected) <= 1e-12 * var_expected);
      CHECK(std::abs(meta.mean.to_host()[0] - double(run_avg)) <= 1e-12);
    }
  }
}

// test_meta.cpp:280-289
TEST_CASE("meta step rejects mismatched dimensions and negative variances") {
  MetaEstimator<> meta(ctx(), 0.01);
  GradientSamplePair<> pair{dv({0.0, 0.0}), dv({0.0, 0.0}), 0.0};
  CHECK_THROWS_AS(meta.step(pair, dv({0.0, 0.0, 0.0}), dv({0.0, 0.0})), std::invalid_argument);
  CHECK_THROWS_AS(meta.step(pair, dv({-1.0, 0.0}), dv({0.0, 0.0})), std::logic_error);
  CHECK_THROWS_AS(MetaEstimator<>(ctx(), 0.0), std::invalid_argument);
}

// test_adam.cpp:15-28 + :51-71 (independent transcription, 1e-12)
TEST_CASE("Adam matches the straight-line transcription") {
  Adam<> adam(ctx(), 0.02, 0.9, 0.999);
  std::mt19937_64 gen(11);
  double m = 0, v = 0;
  for (int t = 1; t <= 100; ++t) {
    const double g = 6.0 * double(gen() >> 11) * 0x1.0p-53 - 3.0;
    const double d = adam.step(dv({g})).to_host()[0];
    m = 0.9 * m + (1.0 - 0.9) * g;
    v = 0.999 * v + (1.0 - 0.999) * g * g;
    const double mh = m / (1.0 - std::pow(0.9, t)), vh = v / (1.0 - std::pow(0.999, t));
    CHECK(d == doctest::Approx(-0.02 * mh / (std::sqrt(vh) + 1e-8)).epsilon(1e-12));
  }
  CHECK_THROWS_AS(Adam<>(ctx(), 0.01, 1.0, 0.999), std::invalid_argument);
}

// rng.hpp:23-25 + the C++ standard's 10000th-output value of mt19937_64
TEST_CASE("device engines reproduce std::mt19937_64") {
  Rng eng(ctx(), {5489});
  const auto raw = eng.raw(10000);
  CHECK(raw.back() == 9981545732273789042ULL);
  std::mt19937_64 host_engine(mg_stream_seed(7, 3));
  Rng s = Rng::stream(ctx(), 7, 3);
  const auto u = s.uniform(1000);
  bool same = true;
  for (double x : u) same &= (x == double(host_engine() >> 11) * 0x1.0p-53);
  CHECK(same);
}

// test_problems.cpp:267-274 and :220-229
TEST_CASE("mini-render: identical albedo gives exactly zero diff") {
  MiniRenderProblem problem(ctx(), 5, 3, 13);
  Rng rng = Rng::stream(ctx(), 74, 0);
  const auto albedo = DeviceVec<double>::Constant(ctx(), 5, 0.4);
  const auto pair = problem.sample_pair(albedo, albedo, rng);
  for (double d : pair.diff.to_host()) CHECK(d == 0.0);
  CHECK(pair.step_sq_norm == 0.0);
  CHECK_THROWS_AS(MiniRenderProblem(ctx(), 8, 1), std::invalid_argument);
  MiniRenderProblem a(ctx(), 8, 4, 42), b(ctx(), 8, 4, 42);
  CHECK(a.target_image().to_host() == b.target_image().to_host());
  for (double t : a.target_image().to_host()) CHECK((t >= 0.2 && t <= 1.0));
}

// harness.cpp:90-200 through the device runner: test_harness.cpp:102-134
TEST_CASE("noiseless scripted run reproduces the hand-computed recurrence") {
  mg_experiment_config cfg;
  mg_config_defaults(&cfg);
  cfg.problem = MG_MULT_NOISE;
  cfg.dim = 1;
  cfg.sigma = 0.0;
  cfg.samples_per_iter = 1;
  cfg.trajectory = MG_TRAJ_SCRIPTED_LINEAR;
  cfg.iterations = 3;
  const auto r = run_replicates(ctx(), cfg, 0, 1, 1);
  REQUIRE(r.records[0].iterations_run == 3);
  const auto& prop = r.series[2];
  const auto& alpha = r.series[6];
  const auto& grad_est = r.series[4];
  const auto& ssn = r.series[9];
  CHECK(prop[0] == 2.0);
  CHECK(alpha[0] == 0.0);
  const double var_prop = 4.0 + (0.1 / 0.19) * (1.0 - 4.0);
  const double alpha1 = var_prop / (var_prop + 5.0 + 1e-30);
  CHECK(ssn[1] == 1.0);
  CHECK(alpha[1] == doctest::Approx(alpha1).epsilon(1e-14));
  CHECK(grad_est[1] == doctest::Approx(1.0).epsilon(1e-14));
}
