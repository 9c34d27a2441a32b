// Device plumbing shared by the metagrad drop-in headers (include/metagrad_gpu/
// metagrad/{moment2,meta,adam}.hpp): a per-thread libmgcuda context and the
// staging of metagrad::Vec arguments through the device.
//
// The reference's estimator objects have value semantics over host vectors
// (moment2.hpp:21-50, meta.hpp:71-114, adam.hpp:14-50) and its tests inject
// state directly (tests/test_meta.cpp:213-218), so the drop-in keeps the
// state in host Vecs and stages it through the device around every call;
// all arithmetic runs in the sm_100a kernels.  Per call: the operands are
// packed into one page-locked block, moved with ONE host-to-device copy into
// one device block (both grow-only, cached per thread), the kernel runs,
// the results come back in one or two copies and one synchronisation.  The
// device-resident path (no staging at all) is the C-ABI's fused update and
// replicate runner (include/mgcuda.h).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "mgcuda.h"
#include "metagrad/vec.hpp"

namespace metagrad_gpu {

// C-ABI status -> the reference's exception types.
inline void check(int status) {
  if (status == MG_OK) return;
  const std::string msg = mg_last_error();
  switch (status) {
    case MG_EINVAL: throw std::invalid_argument(msg);
    case MG_ELOGIC: throw std::logic_error(msg);
    case MG_EDOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error("libmgcuda: " + msg);
  }
}

// Argument validation with the reference's exception type and message.
inline void require(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(what);
}

// Per host thread: one context (device + private stream) and the staging
// blocks.  The reference runs one replicate per std::thread
// (harness.cpp:263-271); a libmgcuda context is single-threaded.
// Device = $MG_DEVICE (default 0).
struct ThreadState {
  mg_ctx* ctx = nullptr;
  void* dev = nullptr;   // device staging block
  void* host = nullptr;  // page-locked host staging block
  size_t cap = 0;        // doubles in each block
  mg_mt64* engine = nullptr;  // one device mt19937_64 (problems.hpp adapters)
  ~ThreadState() {
    if (engine) mg_mt64_destroy(engine);
    if (ctx) {
      if (dev) mg_free(ctx, dev);
      mg_ctx_synchronize(ctx);
      mg_ctx_destroy(ctx);
    }
    if (host) mg_host_free(host);
  }
};

inline ThreadState& thread_state() {
  thread_local ThreadState t;
  if (!t.ctx) {
    const char* dev = std::getenv("MG_DEVICE");
    check(mg_ctx_create(dev ? std::atoi(dev) : 0, nullptr, &t.ctx));
  }
  return t;
}

inline mg_ctx* ctx() { return thread_state().ctx; }

// Device initialisation (CUDA context creation, ~0.1-0.5 s) happens when the
// program loads, not inside the first timed estimator call.  Without a
// device it is deferred: the first call then throws.  MG_LAZY_INIT=1 defers
// it in any case (e.g. for programs that fork before using the estimators).
inline const bool kDeviceInitialised = [] {
  const char* lazy = std::getenv("MG_LAZY_INIT");
  if (lazy && lazy[0] == '1') return false;
  try {
    ctx();
    return true;
  } catch (...) {
    return false;
  }
}();

// One call's operands: `slots` vectors of n doubles, contiguous on the host
// (page-locked) and on the device.
class Call {
 public:
  Call(Eigen::Index n, int slots) : n_(size_t(n > 0 ? n : 0)), t_(thread_state()) {
    const size_t need = n_ * size_t(slots);
    if (need > t_.cap) {
      const size_t cap = std::max(need, 2 * t_.cap);
      if (t_.dev) check(mg_free(t_.ctx, t_.dev));
      if (t_.host) check(mg_host_free(t_.host));
      t_.dev = t_.host = nullptr;
      t_.cap = 0;
      check(mg_malloc(t_.ctx, sizeof(double) * cap, &t_.dev));
      check(mg_host_malloc(sizeof(double) * cap, &t_.host));
      t_.cap = cap;
    }
  }
  double* dev(int slot) const { return static_cast<double*>(t_.dev) + size_t(slot) * n_; }
  double* host(int slot) const { return static_cast<double*>(t_.host) + size_t(slot) * n_; }
  // pack v into slot; returns the slot's device pointer
  double* put(int slot, const metagrad::Vec& v) const {
    if (n_) std::memcpy(host(slot), v.data(), sizeof(double) * n_);
    return dev(slot);
  }
  void upload(int first, int count) const {
    check(mg_copy_async(t_.ctx, dev(first), host(first), sizeof(double) * n_ * size_t(count)));
  }
  void download(int first, int count) const {
    check(mg_copy_async(t_.ctx, host(first), dev(first), sizeof(double) * n_ * size_t(count)));
  }
  void finish() const { check(mg_ctx_synchronize(t_.ctx)); }
  void get(int slot, metagrad::Vec& v) const {
    if (v.size() != Eigen::Index(n_)) v = metagrad::Vec::Zero(Eigen::Index(n_));
    if (n_) std::memcpy(v.data(), host(slot), sizeof(double) * n_);
  }
  metagrad::Vec get(int slot) const {
    metagrad::Vec v = metagrad::Vec::Zero(Eigen::Index(n_));
    get(slot, v);
    return v;
  }

 private:
  size_t n_;
  ThreadState& t_;
};

}  // namespace metagrad_gpu
