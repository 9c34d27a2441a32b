// The per-parameter arithmetic of one fused meta-estimator iteration
// (rows A8-A11), shared by the update kernels (update.cu) and the fused
// sample+update kernels (render.cu).  Every expression follows the reference
// operand order; with --fmad=false the fp64 instantiation is bit-identical
// to the oracle.
#pragma once

#include <math.h>

#include "mg_common.cuh"

namespace mg {

struct MetaK {
  double lr, eps_step, eps_alpha, prop_coef, beta_delta, proj_lo, ssn_host, proj_hi;
  double beta_f = 0.0;
  int clip, diff_norm, project, ssn_from_host;
  int prop_dev = 0;     // 1: prop coefficient from the device power
  int prop_adv = 0;     // 1: advance the device beta_f power (also when beta_f > 0)
};

template <class T>
struct MetaPtrs {
  const T* __restrict__ prop;
  const T* __restrict__ diff;
  const T* __restrict__ vprop;
  const T* __restrict__ vdiff;
  T* __restrict__ m2p;
  T* __restrict__ m2d;
  T* __restrict__ mean;
  T* __restrict__ var;
  T* __restrict__ ap;
  const T* pin;  // may alias pout
  T* pout;
  const T* __restrict__ pprev;
  const T* __restrict__ target;
  T* __restrict__ delta;
};

// Per-launch scalar state, identical in every thread (read once from the
// device scalars written by the previous launch's epilogue).
struct StepScal {
  double ssn, norm, c_diff, dpow, ppow, c_prop;
  int64_t cnt0, cnt;
  bool active;
};

__device__ __forceinline__ StepScal load_step_scalars(const MetaK& k, const mg_update_scalars* sc) {
  StepScal s;
  s.ssn = k.ssn_from_host ? k.ssn_host : __ldcg(&sc->ssn);
  s.active = s.ssn > 0.0;                         // harness.cpp:153
  s.cnt0 = __ldcg(&sc->diff_count);
  s.dpow = __ldcg(&sc->diff_decay_pow);
  s.cnt = s.cnt0;
  if (s.active) {
    s.cnt += 1;                                   // moment2.hpp:34
    s.dpow = s.dpow * k.beta_delta;               // moment2.hpp:35
  }
  s.c_diff = (1.0 - k.beta_delta) / (1.0 - s.dpow);  // moment2.hpp:36-38
  s.norm = sqrt(s.ssn);                           // harness.cpp:154
  // Moment2(beta_f): the host passes (1-b)/(1-b^t) computed by the repeated
  // multiply of moment2.hpp:35, or the device forms the same chain
  s.ppow = __ldcg(&sc->prop_decay_pow);
  if (k.prop_adv || k.beta_f > 0.0) s.ppow = s.ppow * k.beta_f;
  s.c_prop = k.prop_dev ? (1.0 - k.beta_f) / (1.0 - s.ppow) : k.prop_coef;
  return s;
}

// IEEE a / b and sqrt(v) that keep zero operands off the slow path.  The
// compiler's correctly rounded division and square root send a zero dividend
// (FCHK) and a zero radicand (range test) to an out-of-line subroutine; in a
// texture fit most parameters see no sample in an iteration, so prop = diff =
// 0 and the fused update ran 40 % slower (tools/update_size_probe.py).  The
// results are unchanged bit for bit: 0 / b = a * b (a signed zero) for finite
// nonzero b, sqrt(+-0) = +-0.
// (opaque() hides the substituted operand from the compiler, which would
// otherwise see that the quotient is unused when z holds and fold the
// substitution away.)
__device__ __forceinline__ float opaque(float x) {
  float y;
  asm("mov.b32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ double opaque(double x) {
  double y;
  asm("mov.b64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
template <class T>
__device__ __forceinline__ T div_z(T a, T b) {
  const bool z = a == T(0) && isfinite(b) && b != T(0);
  const T q = opaque(z ? T(1) : a) / b;
  return z ? a * b : q;
}
template <class T>
__device__ __forceinline__ T sqrt_z(T v) {
  const bool z = v == T(0);
  const T r = sqrt(opaque(z ? T(1) : v));
  return z ? v : r;
}

// One parameter of the fused meta iteration.  All inputs already loaded.
template <class T, bool FIRST>
__device__ __forceinline__ void meta_elem(const MetaK& k, const StepScal& s, T prop, T diff,
                                          T vprop, T vdiff, T& m2p, T& m2d, T& mean, T& var,
                                          T& ap, T pin, T pprev, T target, bool has_target,
                                          T& pout, T& delta, Acc& acc) {
  // Moment2(beta_f).step(prop): m2 += (w/w_sum) * (x^2 - m2)
  const T m2p_old = FIRST ? T(0) : m2p;
  const T cp = T(s.c_prop);
  m2p = m2p_old + cp * (vprop * vprop - m2p_old);
  // decoupled diff variance (global or per-param norm)
  T m2d_v = s.cnt0 > 0 ? m2d : T(0);
  T var_diff = T(0);
  if (k.diff_norm == MG_DIFF_NORM_PER_PARAM) {
    const T cs = fabs(pin - pprev);                          // harness.cpp:147
    const T tiny = sizeof(T) == 8 ? T(1e-150) : T(1e-37);    // kTinyCoordStep (fp32: FLT_MIN-ish)
    if (s.active) {
      const T x = div_z(vdiff, std_max(cs, tiny));                 // harness.cpp:149
      m2d_v = m2d_v + T(s.c_diff) * (x * x - m2d_v);
    }
    if (s.cnt > 0) var_diff = m2d_v * (cs * cs);             // harness.cpp:150
  } else {
    if (s.active) {
      const T x = div_z(vdiff, T(s.norm));                         // harness.cpp:154
      m2d_v = m2d_v + T(s.c_diff) * (x * x - m2d_v);
    }
    if (s.cnt > 0) var_diff = m2d_v * T(s.ssn);              // meta.hpp:51-53
  }
  m2d = m2d_v;
  // MetaEstimator::step (meta.hpp:103-112)
  T m = (FIRST ? T(0) : mean) + diff;
  T v = (FIRST ? T(0) : var) + var_diff;
  const T a_prev = FIRST ? T(-INFINITY) : ap;
  T al = div_z(m2p, (m2p + v) + T(k.eps_alpha));
  if (k.clip) al = std_min(al, T(1) / (T(2) - a_prev));      // meta.hpp:30-32
  ap = al;
  const T om = T(1) - al;
  m = al * m + om * prop;
  v = (al * al) * v + (om * om) * m2p;
  mean = m;
  var = v;
  delta = div_z(T(-k.lr) * m, sqrt_z(v) + T(k.eps_step));
  // params += delta; project (harness.cpp:186-187, problems.cpp:228)
  T p = pin + delta;
  if (k.project) p = std_max(p, T(k.proj_lo));
  if (k.project == 2) p = std_min(p, T(k.proj_hi));
  pout = p;
  // fused reductions (problems.cpp:206,214,225; harness.cpp:116)
  const double d = double(p - pin);
  acc.ssn += d * d;
  acc.changed += (p != pin) ? 1u : 0u;
  if (has_target) {
    const double e = double(p - target);
    acc.loss += e * e;
  }
  acc.nonfinite += isfinite(p) ? 0u : 1u;
}

}  // namespace mg
