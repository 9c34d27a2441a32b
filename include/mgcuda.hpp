// mgcuda.hpp — header-only C++ adapter over the C-ABI (include/mgcuda.h)
// that mirrors the reference's metagrad hot-path API (value types, same
// method names and argument meaning, same exception types), so reference
// callers switch by changing the namespace and the vector type:
//
//   metagrad (reference, CPU, Eigen)       mgcuda (this adapter, B200)
//   Rng::stream(seed, r)        rng.hpp:23  Rng::stream(ctx, seed, r)
//   Moment2::step(x)        moment2.hpp:30  Moment2::step(x)
//   GradientSamplePair          meta.hpp:20 GradientSamplePair
//   MetaEstimator::step(...)    meta.hpp:90 MetaEstimator::step(...)  (mean/var/alpha_prev public)
//   Adam::step(g)               adam.hpp:23 Adam::step(g)
//   MiniRenderProblem::sample_pair problems.cpp:197  MiniRenderProblem::sample_pair
//   run_single / run_experiment harness.cpp:90/249  run_replicates(...)
//
// Vectors are DeviceVec (device-resident, fp64 by default = parity mode).
// std::invalid_argument / std::logic_error / std::domain_error are thrown
// exactly where the reference throws them (the C-ABI status codes map 1:1).
#pragma once

#include <cstdint>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mgcuda.h"

namespace mgcuda {

inline void check(int status) {
  if (status == MG_OK) return;
  const std::string msg = mg_last_error();
  switch (status) {
    case MG_EINVAL: throw std::invalid_argument(msg);
    case MG_ELOGIC: throw std::logic_error(msg);
    case MG_EDOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error("mgcuda: " + msg);
  }
}

// One device + stream.  Copyable handle (shared ownership).
class Context {
 public:
  Context() = default;  // empty handle
  explicit Context(int device) {
    mg_ctx* h = nullptr;
    check(mg_ctx_create(device, nullptr, &h));
    h_ = std::shared_ptr<mg_ctx>(h, [](mg_ctx* p) { mg_ctx_destroy(p); });
  }
  mg_ctx* get() const { return h_.get(); }
  void synchronize() const { check(mg_ctx_synchronize(get())); }

 private:
  std::shared_ptr<mg_ctx> h_;
};

// Device vector of double (fp64 parity mode) or float (fast mode).
template <class T = double>
class DeviceVec {
 public:
  static constexpr int32_t dtype = sizeof(T) == 8 ? MG_F64 : MG_F32;
  DeviceVec() = default;
  DeviceVec(const Context& ctx, std::int64_t n) : ctx_(ctx), n_(n) {
    void* p = nullptr;
    check(mg_malloc(ctx_.get(), sizeof(T) * size_t(n), &p));
    p_ = std::shared_ptr<T>(static_cast<T*>(p), [c = ctx_](T* q) { mg_free(c.get(), q); });
  }
  static DeviceVec Constant(const Context& ctx, std::int64_t n, double v) {
    DeviceVec d(ctx, n);
    check(mg_fill(ctx.get(), dtype, n, d.data(), v));
    return d;
  }
  static DeviceVec Zero(const Context& ctx, std::int64_t n) { return Constant(ctx, n, 0.0); }
  static DeviceVec from_host(const Context& ctx, const std::vector<T>& h) {
    DeviceVec d(ctx, std::int64_t(h.size()));
    check(mg_copy_to_device(ctx.get(), d.data(), h.data(), sizeof(T) * h.size()));
    return d;
  }
  std::vector<T> to_host() const {
    std::vector<T> h(static_cast<size_t>(n_));
    if (n_) check(mg_copy_to_host(ctx_.get(), h.data(), data(), sizeof(T) * h.size()));
    return h;
  }
  DeviceVec clone() const {
    DeviceVec d(ctx_, n_);
    check(mg_copy_device(ctx_.get(), d.data(), data(), sizeof(T) * size_t(n_)));
    return d;
  }
  std::int64_t size() const { return n_; }
  T* data() const { return p_.get(); }
  const Context& context() const { return ctx_; }

 private:
  Context ctx_{};
  std::int64_t n_ = 0;
  std::shared_ptr<T> p_;
};

// rng.hpp:18-37: a batch of device std::mt19937_64 engines.
class Rng {
 public:
  Rng(const Context& ctx, const std::vector<std::uint64_t>& engine_seeds) : ctx_(ctx) {
    mg_mt64* g = nullptr;
    check(mg_mt64_create(ctx.get(), int32_t(engine_seeds.size()), engine_seeds.data(), &g));
    g_ = std::shared_ptr<mg_mt64>(g, [](mg_mt64* p) { mg_mt64_destroy(p); });
    streams_ = int32_t(engine_seeds.size());
  }
  static Rng stream(const Context& ctx, std::uint64_t base_seed, std::uint64_t replicate) {
    return Rng(ctx, {mg_stream_seed(base_seed, replicate)});
  }
  // n draws per engine, engine-major
  std::vector<double> uniform(std::int64_t n) { return draw<double>(n, 1); }
  std::vector<double> uniform_pos(std::int64_t n) { return draw<double>(n, 2); }
  std::vector<std::uint64_t> raw(std::int64_t n) { return draw<std::uint64_t>(n, 0); }
  mg_mt64* get() const { return g_.get(); }
  int32_t streams() const { return streams_; }

 private:
  template <class U>
  std::vector<U> draw(std::int64_t n, int32_t kind) {
    DeviceVec<double> buf(ctx_, n * streams_);
    check(mg_mt64_draw(ctx_.get(), g_.get(), n, kind, buf.data()));
    std::vector<U> out(size_t(n * streams_));
    check(mg_copy_to_host(ctx_.get(), out.data(), buf.data(), sizeof(U) * out.size()));
    return out;
  }
  Context ctx_;
  std::shared_ptr<mg_mt64> g_;
  int32_t streams_ = 0;
};

// moment2.hpp:21-50
template <class T = double>
class Moment2 {
 public:
  explicit Moment2(const Context& ctx, double decay = 0.9) : ctx_(ctx) {
    if (!(decay >= 0.0 && decay < 1.0))
      throw std::invalid_argument("Moment2: decay must lie in [0, 1)");
    s_ = mg_moment2_scalars{decay, 1.0, 0};
  }
  void step(const DeviceVec<T>& x) {
    if (s_.count == 0 && m2_.size() == 0) m2_ = DeviceVec<T>(ctx_, x.size());
    if (x.size() != m2_.size()) throw std::invalid_argument("Moment2: sample dimension mismatch");
    check(mg_moment2_step(ctx_.get(), DeviceVec<T>::dtype, x.size(), &s_, m2_.data(), x.data()));
  }
  const DeviceVec<T>& m2() const { return m2_; }
  std::int64_t count() const { return s_.count; }
  double decay() const { return s_.decay; }

 private:
  Context ctx_;
  mg_moment2_scalars s_{};
  DeviceVec<T> m2_;
};

template <class T = double>
struct GradientSamplePair {  // meta.hpp:20-24
  DeviceVec<T> prop;
  DeviceVec<T> diff;
  double step_sq_norm = 0.0;
};

// meta.hpp:71-114.  mean/var/alpha_prev are public and injectable.
template <class T = double>
struct MetaEstimator {
  double lr = 0.001;
  double eps_step = 1e-8;
  double eps_alpha = 1e-30;
  bool clip_enabled = true;
  DeviceVec<T> mean, var, alpha_prev;

  explicit MetaEstimator(const Context& ctx, double lr_ = 0.001, double eps_step_ = 1e-8,
                         double eps_alpha_ = 1e-30)
      : lr(lr_), eps_step(eps_step_), eps_alpha(eps_alpha_), ctx_(ctx) {
    if (!(lr > 0.0)) throw std::invalid_argument("MetaEstimator: lr must be positive");
  }

  DeviceVec<T> step(const GradientSamplePair<T>& s, const DeviceVec<T>& var_prop,
                    const DeviceVec<T>& var_diff) {
    const std::int64_t n = s.prop.size();
    const bool first = mean.size() == 0;
    if (first) {
      mean = DeviceVec<T>(ctx_, n);
      var = DeviceVec<T>(ctx_, n);
      alpha_prev = DeviceVec<T>(ctx_, n);
    }
    if (s.diff.size() != n || var_prop.size() != n || var_diff.size() != n || mean.size() != n)
      throw std::invalid_argument("MetaEstimator: dimension mismatch");
    DeviceVec<T> delta(ctx_, n);
    const mg_meta_params p{lr, eps_step, eps_alpha, clip_enabled ? 1 : 0};
    check(mg_meta_step(ctx_.get(), DeviceVec<T>::dtype, n, &p, first ? 1 : 0, mean.data(),
                       var.data(), alpha_prev.data(), s.prop.data(), s.diff.data(),
                       var_prop.data(), var_diff.data(), delta.data()));
    return delta;
  }

 private:
  Context ctx_;
};

// adam.hpp:14-50
template <class T = double>
class Adam {
 public:
  Adam(const Context& ctx, double lr, double beta1 = 0.9, double beta2 = 0.999,
       double eps = 1e-8)
      : ctx_(ctx) {
    if (!(lr > 0.0)) throw std::invalid_argument("Adam: lr must be positive");
    if (!(beta1 >= 0.0 && beta1 < 1.0) || !(beta2 >= 0.0 && beta2 < 1.0))
      throw std::invalid_argument("Adam: betas must lie in [0, 1)");
    s_ = mg_adam_scalars{lr, beta1, beta2, eps, 1.0, 1.0, 0};
  }
  DeviceVec<T> step(const DeviceVec<T>& grad) {
    if (s_.t == 0 && m_.size() == 0) {
      m_ = DeviceVec<T>(ctx_, grad.size());
      v_ = DeviceVec<T>(ctx_, grad.size());
    }
    if (grad.size() != m_.size()) throw std::invalid_argument("Adam: gradient dimension mismatch");
    DeviceVec<T> delta(ctx_, grad.size());
    check(mg_adam_step(ctx_.get(), DeviceVec<T>::dtype, grad.size(), &s_, m_.data(), v_.data(),
                       grad.data(), delta.data()));
    return delta;
  }
  std::int64_t t() const { return s_.t; }
  const DeviceVec<T>& m() const { return m_; }
  const DeviceVec<T>& v() const { return v_; }
  double beta1_pow() const { return s_.beta1_pow; }
  double beta2_pow() const { return s_.beta2_pow; }

 private:
  Context ctx_;
  mg_adam_scalars s_{};
  DeviceVec<T> m_, v_;
};

// problems.hpp:157-195 / problems.cpp:162-228
class MiniRenderProblem {
 public:
  MiniRenderProblem(const Context& ctx, int pixel_count, int spp, std::uint64_t gen_seed = 1234,
                    double albedo_init = 0.1, double exponent_max = 4.0)
      : ctx_(ctx), pixel_count_(pixel_count), spp_(spp), albedo_init_(albedo_init) {
    if (pixel_count < 1) throw std::invalid_argument("mini-render: pixel_count must be >= 1");
    if (spp < 2) throw std::invalid_argument("mini-render: spp must be at least 2");
    if (!(exponent_max >= 0.0))
      throw std::invalid_argument("mini-render: exponent_max must be >= 0");
    exponents_ = DeviceVec<double>(ctx, pixel_count);
    target_ = DeviceVec<double>(ctx, pixel_count);
    check(mg_minirender_generate(ctx.get(), pixel_count, gen_seed, exponent_max,
                                 exponents_.data(), target_.data()));
  }
  std::string name() const { return "mini-render"; }
  std::int64_t dim() const { return pixel_count_; }
  std::int64_t draws_per_sample() const { return std::int64_t(pixel_count_) * spp_; }
  DeviceVec<double> initial_params() const {
    return DeviceVec<double>::Constant(ctx_, pixel_count_, albedo_init_);
  }
  const DeviceVec<double>& target_image() const { return target_; }
  const DeviceVec<double>& shape_exponents() const { return exponents_; }

  template <class T>
  GradientSamplePair<T> sample_pair(const DeviceVec<T>& now, const DeviceVec<T>& prev,
                                    Rng& rng) const {
    if (now.size() != pixel_count_ || prev.size() != pixel_count_)
      throw std::invalid_argument("mini-render: parameter dimension mismatch");
    GradientSamplePair<T> pair{DeviceVec<T>(ctx_, pixel_count_), DeviceVec<T>(ctx_, pixel_count_),
                               0.0};
    DeviceVec<double> ssn(ctx_, 1);
    check(mg_minirender_sample_pair(ctx_.get(), DeviceVec<T>::dtype, 1, pixel_count_, spp_,
                                    exponents_.data(), target_.data(), rng.get(), now.data(),
                                    prev.data(), pair.prop.data(), pair.diff.data(), ssn.data()));
    pair.step_sq_norm = ssn.to_host()[0];
    return pair;
  }

 private:
  Context ctx_;
  int pixel_count_, spp_;
  double albedo_init_;
  DeviceVec<double> exponents_, target_;
};

// harness.cpp:90-272 on the device: replicates [begin, begin+count) of cfg.
struct ReplicateResult {
  std::vector<mg_run_record> records;
  std::vector<std::vector<double>> series;  // [SERIES][count*iterations]
  std::vector<double> final_params;         // [count][dim]
};

inline ReplicateResult run_replicates(const Context& ctx, const mg_experiment_config& cfg,
                                      int32_t begin, int32_t count, int dim) {
  ReplicateResult r;
  r.records.resize(size_t(count));
  r.series.assign(11, std::vector<double>(size_t(count) * size_t(cfg.iterations)));
  r.final_params.resize(size_t(count) * size_t(dim));
  mg_run_series s{r.series[0].data(), r.series[1].data(), r.series[2].data(), r.series[3].data(),
                  r.series[4].data(), r.series[5].data(), r.series[6].data(), r.series[7].data(),
                  r.series[8].data(), r.series[9].data(), r.series[10].data()};
  check(mg_run_replicates(ctx.get(), &cfg, begin, count, r.records.data(), &s,
                          r.final_params.data()));
  return r;
}

}  // namespace mgcuda
