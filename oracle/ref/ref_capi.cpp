// extern "C" shim over the UNMODIFIED reference library (built from
// /root/reference/proj/src by oracle/ref/Makefile into oracle/_ref/).
//
// TEST INFRASTRUCTURE ONLY.  Used by (a) oracle/gen_golden.py to produce the
// committed golden fixtures under tests/golden/, (b) the -m "not gpu" tests
// that pin the C restatement (oracle/metagrad_oracle.c) against the real
// reference, and (c) bench.py's cpu_baseline / --impl reference legs, which
// time the reference's own CPU code.  Never linked into the product.
//
// Every entry point drives the reference's public API exactly as its own
// harness/tests do; the file:line cited on each is the reference code run.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <json.hpp>

#include "metagrad/adam.hpp"
#include "metagrad/harness.hpp"
#include "metagrad/meta.hpp"
#include "metagrad/moment2.hpp"
#include "metagrad/problems.hpp"
#include "metagrad/rng.hpp"
#include "metagrad/validation.hpp"

using namespace metagrad;

namespace {

Vec to_vec(const double* p, std::int64_t n) {
  Vec v(n);
  for (std::int64_t i = 0; i < n; ++i) v[i] = p[i];
  return v;
}

void from_vec(const Vec& v, double* out) {
  if (!out) return;
  for (Eigen::Index i = 0; i < v.size(); ++i) out[i] = v[i];
}

thread_local std::string g_err;

// "key=value;key=value" -> ExperimentConfig (field names as in
// proj/include/metagrad/harness.hpp:18-67).
ExperimentConfig parse_config(const char* text) {
  ExperimentConfig cfg;
  std::stringstream ss(text ? text : "");
  std::string item;
  while (std::getline(ss, item, ';')) {
    if (item.empty()) continue;
    const auto eq = item.find('=');
    if (eq == std::string::npos) throw std::invalid_argument("bad config item: " + item);
    const std::string k = item.substr(0, eq), v = item.substr(eq + 1);
    auto b = [&] { return v == "1" || v == "true"; };
    if (k == "problem") cfg.problem = v;
    else if (k == "optimizer") cfg.optimizer = v;
    else if (k == "iterations") cfg.iterations = std::stoi(v);
    else if (k == "replicates") cfg.replicates = std::stoi(v);
    else if (k == "seed") cfg.seed = std::stoull(v);
    else if (k == "lr") cfg.lr = std::stod(v);
    else if (k == "beta_f") cfg.beta_f = std::stod(v);
    else if (k == "beta_delta") cfg.beta_delta = std::stod(v);
    else if (k == "beta1") cfg.beta1 = std::stod(v);
    else if (k == "beta2") cfg.beta2 = std::stod(v);
    else if (k == "eps_step") cfg.eps_step = std::stod(v);
    else if (k == "eps_alpha") cfg.eps_alpha = std::stod(v);
    else if (k == "adam_eps") cfg.adam_eps = std::stod(v);
    else if (k == "dim") cfg.dim = std::stoi(v);
    else if (k == "sigma") cfg.sigma = std::stod(v);
    else if (k == "samples_per_iter") cfg.samples_per_iter = std::stoi(v);
    else if (k == "target_mean") cfg.target_mean = std::stod(v);
    else if (k == "rate_init") cfg.rate_init = std::stod(v);
    else if (k == "pixel_count") cfg.pixel_count = std::stoi(v);
    else if (k == "spp") cfg.spp = std::stoi(v);
    else if (k == "problem_seed") cfg.problem_seed = std::stoull(v);
    else if (k == "albedo_init") cfg.albedo_init = std::stod(v);
    else if (k == "exponent_max") cfg.exponent_max = std::stod(v);
    else if (k == "trajectory") cfg.trajectory = v;
    else if (k == "traj_rate") cfg.traj_rate = std::stod(v);
    else if (k == "no_alpha_clip") cfg.no_alpha_clip = b();
    else if (k == "independent_variance_samples") cfg.independent_variance_samples = b();
    else if (k == "diff_norm") cfg.diff_norm = v;
    else if (k == "coord") cfg.coord = std::stoi(v);
    else if (k == "converge_threshold") cfg.converge_threshold = std::stod(v);
    else if (k == "threads") cfg.threads = std::stoi(v);
    else throw std::invalid_argument("unknown config key: " + k);
  }
  return cfg;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {  // includes domain_error
    g_err = e.what();
    return dynamic_cast<const std::domain_error*>(&e) ? 3 : 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// rng.hpp:9-14
std::uint64_t ref_mix64(std::uint64_t x) { return mix64(x); }

// rng.hpp:20 (Rng(seed)) or rng.hpp:23-25 (Rng::stream) raw / uniform output.
// mode: 0 = Rng(seed).raw(), 1 = stream(seed, rep).raw(), 2 = stream.uniform(),
//       3 = stream.uniform_pos(), 4 = Rng(seed).uniform()
void ref_rng_draws(std::uint64_t seed, std::uint64_t rep, int mode, std::int64_t n, void* out) {
  Rng rng = (mode == 0 || mode == 4) ? Rng(seed) : Rng::stream(seed, rep);
  auto* u = static_cast<std::uint64_t*>(out);
  auto* d = static_cast<double*>(out);
  for (std::int64_t i = 0; i < n; ++i) {
    switch (mode) {
      case 0: case 1: u[i] = rng.raw(); break;
      case 2: case 4: d[i] = rng.uniform(); break;
      default: d[i] = rng.uniform_pos(); break;
    }
  }
}

// problems.cpp:162-173
int ref_minirender_gen(int pixel_count, int spp, std::uint64_t gen_seed, double albedo_init,
                       double exponent_max, double* out_b, double* out_T, double* out_init) {
  return guarded([&] {
    MiniRenderProblem p(pixel_count, spp, gen_seed, albedo_init, exponent_max);
    from_vec(p.shape_exponents(), out_b);
    from_vec(p.target_image(), out_T);
    from_vec(p.initial_params(), out_init);
  });
}

// problems.cpp:177-195 on caller-supplied uniforms
int ref_minirender_kernel_terms(int pixel_count, int spp, std::uint64_t gen_seed,
                                double exponent_max, const double* uniforms, double* out_cross,
                                double* out_mean_basis) {
  return guarded([&] {
    MiniRenderProblem p(pixel_count, spp, gen_seed, 0.1, exponent_max);
    std::vector<double> u(uniforms, uniforms + static_cast<std::size_t>(pixel_count) * spp);
    const auto t = p.kernel_terms(u);
    from_vec(t.cross, out_cross);
    from_vec(t.mean_basis, out_mean_basis);
  });
}

// problems.cpp:197-217; the Rng is Rng::stream(seed, rep) advanced by `skip`
// sample_pair calls first (so consecutive iterations can be reproduced).
int ref_minirender_sample_pair(int pixel_count, int spp, std::uint64_t gen_seed,
                               double exponent_max, const double* now, const double* prev,
                               std::uint64_t seed, std::uint64_t rep, int skip, double* out_prop,
                               double* out_diff, double* out_ssn) {
  return guarded([&] {
    MiniRenderProblem p(pixel_count, spp, gen_seed, 0.1, exponent_max);
    Rng rng = Rng::stream(seed, rep);
    const Vec a = to_vec(now, pixel_count), b = to_vec(prev, pixel_count);
    for (int s = 0; s < skip; ++s) p.sample_pair(a, b, rng);
    const auto pair = p.sample_pair(a, b, rng);
    from_vec(pair.prop, out_prop);
    from_vec(pair.diff, out_diff);
    *out_ssn = pair.step_sq_norm;
  });
}

// problems.cpp:54-76
int ref_exprate_sample_pair(double target_mean, int samples_per_iter, double rate_now,
                            double rate_prev, std::uint64_t seed, std::uint64_t rep, int skip,
                            double* out_prop, double* out_diff, double* out_ssn) {
  return guarded([&] {
    ExpRateProblem p(target_mean, samples_per_iter, 2.0);
    Rng rng = Rng::stream(seed, rep);
    const Vec a = Vec::Constant(1, rate_now), b = Vec::Constant(1, rate_prev);
    for (int s = 0; s < skip; ++s) p.sample_pair(a, b, rng);
    const auto pair = p.sample_pair(a, b, rng);
    *out_prop = pair.prop[0];
    *out_diff = pair.diff[0];
    *out_ssn = pair.step_sq_norm;
  });
}

// problems.cpp:121-139 (target = 0 as make_problem builds it, harness.cpp:71-73)
int ref_multnoise_sample_pair(int dim, double sigma, int samples_per_iter, const double* target,
                              const double* now, const double* prev, std::uint64_t seed,
                              std::uint64_t rep, int skip, double* out_prop, double* out_diff,
                              double* out_ssn) {
  return guarded([&] {
    MultNoiseQuadratic p(to_vec(target, dim), sigma, samples_per_iter);
    Rng rng = Rng::stream(seed, rep);
    const Vec a = to_vec(now, dim), b = to_vec(prev, dim);
    for (int s = 0; s < skip; ++s) p.sample_pair(a, b, rng);
    const auto pair = p.sample_pair(a, b, rng);
    from_vec(pair.prop, out_prop);
    from_vec(pair.diff, out_diff);
    *out_ssn = pair.step_sq_norm;
  });
}

// moment2.hpp:30-39, `steps` consecutive steps over rows of xs[steps][n];
// m2 after every step written to out[steps][n].
int ref_moment2_run(double decay, std::int64_t n, int steps, const double* xs, double* out) {
  return guarded([&] {
    Moment2 m(decay);
    for (int s = 0; s < steps; ++s) {
      m.step(to_vec(xs + static_cast<std::size_t>(s) * n, n));
      from_vec(m.m2(), out + static_cast<std::size_t>(s) * n);
    }
  });
}

// meta.hpp:90-113 with injected state (as tests/test_meta.cpp:213-218 does).
// has_state = 0 starts from the lazy-init state (mean=0, var=0, alpha=-inf).
int ref_meta_step(std::int64_t n, double lr, double eps_step, double eps_alpha, int clip,
                  int has_state, double* mean, double* var, double* alpha_prev, const double* prop,
                  const double* diff, double ssn, const double* var_prop, const double* var_diff,
                  double* out_delta) {
  return guarded([&] {
    MetaEstimator meta(lr, eps_step, eps_alpha);
    meta.clip_enabled = clip != 0;
    if (has_state) {
      meta.mean = to_vec(mean, n);
      meta.var = to_vec(var, n);
      meta.alpha_prev = to_vec(alpha_prev, n);
    }
    GradientSamplePair pair{to_vec(prop, n), to_vec(diff, n), ssn};
    const Vec d = meta.step(pair, to_vec(var_prop, n), to_vec(var_diff, n));
    from_vec(meta.mean, mean);
    from_vec(meta.var, var);
    from_vec(meta.alpha_prev, alpha_prev);
    from_vec(d, out_delta);
  });
}

// adam.hpp:23-37, `steps` steps over grads[steps][n]; m, v, delta after the
// last step.
int ref_adam_run(std::int64_t n, int steps, double lr, double beta1, double beta2, double eps,
                 const double* grads, double* out_m, double* out_v, double* out_delta) {
  return guarded([&] {
    Adam adam(lr, beta1, beta2, eps);
    Vec d;
    for (int s = 0; s < steps; ++s) d = adam.step(to_vec(grads + static_cast<std::size_t>(s) * n, n));
    from_vec(adam.m(), out_m);
    from_vec(adam.v(), out_v);
    from_vec(d, out_delta);
  });
}

// harness.cpp:90-200.  Fills caller buffers of iterations*dim (vectors) or
// iterations (scalars); any may be null.  Returns the status code
// (0 completed, 1 converged, 2 diverged) in *out_status.
int ref_run_single(const char* cfg_text, int replicate, int* out_iters, int* out_status,
                   std::int64_t* out_draws, std::int64_t* out_evals, double* params, double* loss,
                   double* prop, double* diff, double* ssn, double* mean_est, double* var_est,
                   double* alpha, double* delta, double* true_grad) {
  return guarded([&] {
    const ExperimentConfig cfg = parse_config(cfg_text);
    const RunRecord rec = run_single(cfg, replicate);
    *out_iters = rec.iterations_run;
    *out_status = static_cast<int>(rec.status);
    *out_draws = rec.draws_used;
    *out_evals = rec.evals_used;
    const std::size_t dim = rec.params.empty() ? 0 : static_cast<std::size_t>(rec.params[0].size());
    for (int i = 0; i < rec.iterations_run; ++i) {
      const auto k = static_cast<std::size_t>(i);
      if (params) from_vec(rec.params[k], params + k * dim);
      if (loss) loss[k] = rec.loss[k];
      if (prop) from_vec(rec.prop[k], prop + k * dim);
      if (diff) from_vec(rec.diff[k], diff + k * dim);
      if (ssn) ssn[k] = rec.step_sq_norm[k];
      if (mean_est) from_vec(rec.mean_est[k], mean_est + k * dim);
      if (var_est) from_vec(rec.var_est[k], var_est + k * dim);
      if (alpha && !rec.alpha.empty()) from_vec(rec.alpha[k], alpha + k * dim);
      if (delta) from_vec(rec.delta[k], delta + k * dim);
      if (true_grad) from_vec(rec.true_grad[k], true_grad + k * dim);
    }
  });
}

// harness.cpp:249-302 (+ writers :311-342).  Returns the wall time in
// seconds of run_experiment; writes the aggregate CSV to csv_path if given.
static void write_text(const char* path, const std::string& text) {
  FILE* f = std::fopen(path, "wb");
  if (!f) throw std::runtime_error(std::string("cannot open output file: ") + path);
  std::fwrite(text.data(), 1, text.size(), f);
  std::fclose(f);
}

// run_experiment + every writer of harness.cpp:305-427: the aggregate CSV,
// summary_json, and write_replicate_csv of replicate `rep_index` (paths may
// be NULL/empty to skip).  Golden for tests/test_report_format.py.
int ref_run_experiment_outputs(const char* cfg_text, const char* csv_path, const char* json_path,
                               const char* rep_csv_path, int rep_index) {
  return guarded([&] {
    const ExperimentConfig cfg = parse_config(cfg_text);
    const AggregateReport rep = run_experiment(cfg);
    if (csv_path && *csv_path) {
      std::ostringstream os;
      write_aggregate_csv(rep, os);
      write_text(csv_path, os.str());
    }
    if (json_path && *json_path) write_text(json_path, summary_json(rep));
    if (rep_csv_path && *rep_csv_path) {
      if (rep_index < 0 || rep_index >= int(rep.records.size()))
        throw std::invalid_argument("replicate index out of range");
      std::ostringstream os;
      write_replicate_csv(rep.records[size_t(rep_index)], os);
      write_text(rep_csv_path, os.str());
    }
  });
}

int ref_run_experiment(const char* cfg_text, const char* csv_path, double* out_seconds,
                       int* out_diverged) {
  return guarded([&] {
    const ExperimentConfig cfg = parse_config(cfg_text);
    const auto t0 = std::chrono::steady_clock::now();
    const AggregateReport rep = run_experiment(cfg);
    *out_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (out_diverged) *out_diverged = rep.diverged_count;
    if (csv_path && *csv_path) {
      // harness.cpp:311-334 into a string, then plain stdio (std::ofstream
      // crashes when numpy's bundled runtime is loaded in the same process)
      std::ostringstream os;
      write_aggregate_csv(rep, os);
      const std::string text = os.str();
      FILE* f = std::fopen(csv_path, "wb");
      if (!f) throw std::runtime_error(std::string("cannot open output file: ") + csv_path);
      std::fwrite(text.data(), 1, text.size(), f);
      std::fclose(f);
    }
  });
}

// One meta-estimator update step of the reference harness (harness.cpp:
// 275-291 + 317-318): Moment2(beta_f).step(prop); global-mode decoupled
// diff EMA; MetaEstimator::step; params += delta.  Runs `steps` steps over a
// vector of n parameters split into `threads` independent contiguous chunks
// (each chunk its own estimator objects on its own std::thread; the update
// is elementwise, so chunking is exact except for the global ssn, which is
// given).  Inputs cycle over `pool` (prop, diff) batches of n doubles each.
// The first `warmup` steps are untimed; returns the mean seconds per timed
// step in *out_sec_per_step and the median in *out_median (may be null).
int ref_meta_update_bench(std::int64_t n, int warmup, int steps, int threads, int pool,
                          const double* props, const double* diffs, double ssn,
                          double* out_sec_per_step, double* out_median) {
  return guarded([&] {
    const int T = threads < 1 ? 1 : threads;
    struct Chunk {
      std::int64_t lo, hi;
      Moment2 mp{0.9}, md{0.5};
      MetaEstimator meta{0.01};
      Vec params;
    };
    std::vector<Chunk> chunks(static_cast<std::size_t>(T));
    for (int t = 0; t < T; ++t) {
      chunks[t].lo = n * t / T;
      chunks[t].hi = n * (t + 1) / T;
      chunks[t].params = Vec::Zero(chunks[t].hi - chunks[t].lo);
    }
    std::vector<double> times;
    for (int s = 0; s < warmup + steps; ++s) {
      const double* P = props + static_cast<std::size_t>(s % pool) * n;
      const double* D = diffs + static_cast<std::size_t>(s % pool) * n;
      const double step_ssn = s == 0 ? 0.0 : ssn;
      const auto t0 = std::chrono::steady_clock::now();
      auto work = [&](Chunk& c) {
        const std::int64_t m = c.hi - c.lo;
        GradientSamplePair pair{to_vec(P + c.lo, m), s == 0 ? Vec(Vec::Zero(m)) : to_vec(D + c.lo, m),
                                step_ssn};
        c.mp.step(pair.prop);
        if (pair.step_sq_norm > 0.0) c.md.step(pair.diff / std::sqrt(pair.step_sq_norm));
        const Vec var_diff = c.md.count() > 0 ? rescale_diff_variance(c.md.m2(), pair.step_sq_norm)
                                              : Vec(Vec::Zero(m));
        const Vec delta = c.meta.step(pair, c.mp.m2(), var_diff);
        c.params += delta;
      };
      if (T == 1) {
        work(chunks[0]);
      } else {
        std::vector<std::thread> ws;
        for (auto& c : chunks) ws.emplace_back([&work, &c] { work(c); });
        for (auto& w : ws) w.join();
      }
      if (s >= warmup)
        times.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    if (times.empty()) throw std::invalid_argument("ref_meta_update_bench: no timed step");
    double sum = 0.0;
    for (double x : times) sum += x;
    *out_sec_per_step = sum / double(times.size());
    std::sort(times.begin(), times.end());
    if (out_median) *out_median = times[times.size() / 2];
  });
}

// harness.cpp:305-309 (shortest round-trip std::to_chars)
int ref_format_double(double v, char* out, int cap) {
  const std::string s = format_double(v);
  if (int(s.size()) + 1 > cap) return 1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}

// A double as the reference's summary_json emits it (nlohmann::json dump,
// harness.cpp:367-427) — pins report.json_double.
int ref_json_double(double v, char* out, int cap) {
  const std::string s = nlohmann::ordered_json(v).dump();
  if (int(s.size()) + 1 > cap) return 1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}

// validation.cpp:262-299
int ref_validation_suite(std::uint64_t seed, int* out_passed, int* out_total) {
  return guarded([&] {
    const auto results = run_validation_suite(seed);
    int ok = 0;
    for (const auto& r : results) ok += r.pass ? 1 : 0;
    *out_passed = ok;
    *out_total = static_cast<int>(results.size());
  });
}

}  // extern "C"
