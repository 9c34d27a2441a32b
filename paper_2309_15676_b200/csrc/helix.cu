// F1 slice 2 (BASELINE.json configs[2]): a procedural helix of 64 spheres on
// a diffuse ground plane, lit by a rectangular area light and a constant
// environment, path traced to depth 4 with next-event estimation; the spheres
// share one principled-style BSDF (Lambert + GGX/Schlick/Smith) whose 5
// global parameters (base RGB, metalness, roughness) are optimised.
// Scene, sampling and estimators: DESIGN.md §F1b; CPU oracle:
// oracle/metagrad_oracle.c mgo_helix_* (the reference has no renderer).
//
// One thread per pixel traces three paths (Philox counter = pixel,
// iteration, path, vertex slot).  Directions are cosine-sampled (Malley,
// rejection in the unit disk) independently of the parameters, so
//   * the parameter derivative rides along the path in forward mode
//     (beta, d beta/d theta per colour channel), and
//   * the finite-difference sample evaluates the SAME path (shared primary
//     hit, bounces and shadow rays) at theta_t and theta_{t-1}.
// Sphere data sits in shared memory (broadcast reads); the 5+5 gradient sums
// are reduced exactly in 2^-40 fixed point (warp shuffles, one int64 atomic
// per CTA and parameter), so the result is deterministic and bit-identical to
// the oracle in fp64.
#include <math.h>

#include "mg_common.cuh"
#include "philox.cuh"

namespace mg {
// mg_set_option("helix_split", 0): the one-kernel sample pair instead of
// the path / combine stages (defined in the fp64 translation unit)
extern bool g_helix_split;
#ifndef MG_HELIX_F32_TU
bool g_helix_split = true;
#endif
namespace {

constexpr int kHThreads = 128;
constexpr int kMaxV = 4;
constexpr int kNP = 5;
constexpr int kMaxSph = 256;
constexpr double kEps = 1e-4, kTanH = 0.35, kLY = 4.0, kLA = 4.0;
constexpr double kPiH = 3.14159265358979323846;
constexpr double kFixH = 1099511627776.0;  // 2^40

struct HelixK {
  int W, H, nsph;
  int row0, row1;  // image rows [row0, row1) of this tile (sample pairs)
  double Le[3], env[3], ground[3];
  uint64_t key;
  uint32_t iteration;
  const uint32_t* it_offset;  // device iteration offset or null (mg_ctx_set_iteration_offset)
};

template <class T>
struct V3 {
  T x, y, z;
};

template <class T>
__device__ __forceinline__ T dot3(const V3<T>& a, const V3<T>& b) {
  return (a.x * b.x + a.y * b.y) + a.z * b.z;
}

__device__ __forceinline__ void hrng(uint64_t key, uint32_t pix, uint32_t it, uint32_t path,
                                     uint32_t slot, double u[4]) {
  const Philox4 r =
      philox4x32_10(Philox4{{pix, it, path, slot}}, uint32_t(key), uint32_t(key >> 32));
#pragma unroll
  for (int k = 0; k < 4; ++k) u[k] = double(r.x[k]) * 0x1.0p-32;
}

// closest hit: 0 none, 1 sphere, 2 ground, 3 light (camera rays only)
template <class T>
__device__ int intersect(const T* __restrict__ sph, int nsph, const V3<T>& o, const V3<T>& d,
                         bool want_light, T tmax, T& t_out, int& k_out) {
  T best = tmax;
  int kind = 0, kb = -1;
  for (int k = 0; k < nsph; ++k) {
    const T* c = sph + 4 * k;
    const V3<T> oc{o.x - c[0], o.y - c[1], o.z - c[2]};
    const T b = dot3(oc, d);
    const T cc = dot3(oc, oc) - c[3] * c[3];
    T t;
    if constexpr (sizeof(T) == 8) {  // the oracle's expression order (parity)
      const T disc = b * b - cc;
      if (disc < T(0)) continue;
      const T sq = sqrt(disc);
      t = -b - sq;
      if (t < T(kEps)) t = -b + sq;
    } else {
      // fp32: b*b - cc cancels for a distant sphere (|oc|^2 ~ 36 vs r^2 =
      // 0.01), leaving ~1e-5 error in t and ~1e-4 in the normal, which the
      // GGX lobe amplifies.  Discriminant from the ray's closest approach
      // (r^2 - |oc - b d|^2) and the cancellation-free pair of roots q,
      // cc / q instead.
      // cheap reject first: the cancelling form is off by at most a few
      // ulp of b^2 (+ |oc|^2), so a clear miss stays a miss
      if (b * b - cc < T(-1e-6) * (b * b + dot3(oc, oc))) continue;
      const V3<T> f{oc.x - b * d.x, oc.y - b * d.y, oc.z - b * d.z};
      const T disc = c[3] * c[3] - dot3(f, f);
      if (disc < T(0)) continue;
      const T qq = -b - copysign(sqrt(disc), b);
      if (qq == T(0)) continue;
      const T r0 = cc / qq;
      const T t0 = fmin(qq, r0), t1 = fmax(qq, r0);
      t = t0 < T(kEps) ? t1 : t0;
    }
    if (t < T(kEps) || t >= best) continue;
    best = t;
    kind = 1;
    kb = k;
  }
  if (d.y < T(0)) {
    const T t = -o.y / d.y;
    if (t >= T(kEps) && t < best) {
      best = t;
      kind = 2;
    }
  }
  if (want_light && d.y > T(0)) {
    const T t = (T(kLY) - o.y) / d.y;
    if (t >= T(kEps) && t < best) {
      const T x = o.x + t * d.x, z = o.z + t * d.z;
      if (x >= T(-1) && x <= T(1) && z >= T(-1) && z <= T(1)) {
        best = t;
        kind = 3;
      }
    }
  }
  t_out = best;
  k_out = kb;
  return kind;
}

// principled BSDF f[c] and its non-zero derivatives df[c][k], k = 0: d/d base_c
// (base_c' != c does not enter f_c), 1: d/d metal, 2: d/d rough
template <class T>
__device__ __forceinline__ void bsdf(const T* th, const V3<T>& n, const V3<T>& wi,
                                     const V3<T>& wo, T f[3], T df[3][3]) {
  const T metal = th[3], rough = th[4];
  const T alpha = T(0.05) + T(0.95) * (rough * rough);
  const T a2 = alpha * alpha;
  V3<T> h{wi.x + wo.x, wi.y + wo.y, wi.z + wo.z};
  const T hl = sqrt(dot3(h, h));
  h.x /= hl;
  h.y /= hl;
  h.z /= hl;
  const T nh = dot3(n, h), ni = dot3(n, wi), no = dot3(n, wo), ih = dot3(wi, h);
  const T den = nh * nh * (a2 - T(1)) + T(1);
  const T D = a2 / (T(kPiH) * (den * den));
  const T dD_da2 = (den - T(2) * a2 * (nh * nh)) / (T(kPiH) * ((den * den) * den));
  const T si = sqrt(a2 + (T(1) - a2) * (ni * ni));
  const T so = sqrt(a2 + (T(1) - a2) * (no * no));
  const T G1i = (T(2) * ni) / (ni + si), G1o = (T(2) * no) / (no + so);
  const T dG1i = ((T(-2) * ni) / ((ni + si) * (ni + si))) * ((T(1) - ni * ni) / (T(2) * si));
  const T dG1o = ((T(-2) * no) / ((no + so) * (no + so))) * ((T(1) - no * no) / (T(2) * so));
  const T G = G1i * G1o;
  const T dG_da2 = dG1i * G1o + G1i * dG1o;
  const T q = T(1) - ih;
  const T q5 = ((q * q) * (q * q)) * q;
  const T denom = T(4) * ni * no;
  const T DG = (D * G) / denom;
  const T dDG_drough = (((dD_da2 * G + D * dG_da2) / denom) * (T(2) * alpha)) * (T(1.9) * rough);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const T base = th[c];
    const T F0 = T(0.04) * (T(1) - metal) + base * metal;
    const T F = F0 + (T(1) - F0) * q5;
    f[c] = ((T(1) - metal) * base) / T(kPiH) + DG * F;
    df[c][0] = (T(1) - metal) / T(kPiH) + DG * (metal * (T(1) - q5));
    df[c][1] = (-base) / T(kPiH) + DG * ((base - T(0.04)) * (T(1) - q5));
    df[c][2] = dDG_drough * F;
  }
}

// One path evaluated for NSETS parameter sets: radiance L[s][c] and its
// non-zero derivatives dL[s][c][k] (k: base_c, metal, rough — radiance of
// channel c depends on no other channel's base colour, so the other
// entries of d L_c / d theta are exactly zero and are not carried).
constexpr int kND = 3;
// inlined into the path kernels (out of line: an ABI call with a 304-byte
// stack frame; inlined fp32 141 registers, no spills): configs[2] fp32
// 0.175 -> 0.153 ms, fp64 0.299 -> 0.235 ms per iteration
#ifndef MG_HELIX_INLINE
#define MG_HELIX_INLINE 1
#endif
#if MG_HELIX_INLINE
#define MG_HELIX_TRACE __device__ __forceinline__
#else
#define MG_HELIX_TRACE __device__ __noinline__
#endif
template <class T, int NSETS>
MG_HELIX_TRACE void trace(const HelixK& q, const T* __restrict__ sph, const T (&th)[2][kNP], int px,
                      int py, uint32_t path, T L[NSETS][3], T dL[NSETS][3][kND]) {
  const uint32_t pix = uint32_t(py * q.W + px);
  double u[4];
  hrng(q.key, pix, q.iteration, path, 0u, u);
  const T sx = T(((double(px) + u[0]) / double(q.W)) * 2.0 - 1.0);
  const T sy = T(1.0 - ((double(py) + u[1]) / double(q.H)) * 2.0);
  V3<T> o{T(0), T(1), T(6)};
  V3<T> d{sx * T(kTanH) * T(double(q.W) / double(q.H)), sy * T(kTanH), T(-1)};
  const T dl = sqrt(dot3(d, d));
  d.x /= dl;
  d.y /= dl;
  d.z /= dl;
  T beta[NSETS][3], dbeta[NSETS][3][kND];
#pragma unroll
  for (int s = 0; s < NSETS; ++s)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      beta[s][c] = T(1);
      L[s][c] = T(0);
#pragma unroll
      for (int k = 0; k < kND; ++k) {
        dbeta[s][c][k] = T(0);
        dL[s][c][k] = T(0);
      }
    }
  for (int v = 0; v < kMaxV; ++v) {
    T t;
    int kk;
    const int kind = intersect<T>(sph, q.nsph, o, d, v == 0, T(1e30), t, kk);
    if (kind == 0) {
#pragma unroll
      for (int s = 0; s < NSETS; ++s)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          L[s][c] += beta[s][c] * T(q.env[c]);
#pragma unroll
          for (int j = 0; j < kND; ++j) dL[s][c][j] += dbeta[s][c][j] * T(q.env[c]);
        }
      return;
    }
    if (kind == 3) {
#pragma unroll
      for (int s = 0; s < NSETS; ++s)
#pragma unroll
        for (int c = 0; c < 3; ++c) L[s][c] += T(q.Le[c]);
      return;
    }
    const V3<T> x{o.x + t * d.x, o.y + t * d.y, o.z + t * d.z};
    V3<T> n;
    if (kind == 1) {
      const T* c = sph + 4 * kk;
      n = V3<T>{(x.x - c[0]) / c[3], (x.y - c[1]) / c[3], (x.z - c[2]) / c[3]};
    } else {
      n = V3<T>{T(0), T(1), T(0)};
    }
    const V3<T> wo{-d.x, -d.y, -d.z};
    hrng(q.key, pix, q.iteration, path, uint32_t(v * 256 + 1), u);
    // next-event estimation to the area light
    const V3<T> ly{T(-1.0 + 2.0 * u[0]), T(kLY), T(-1.0 + 2.0 * u[1])};
    V3<T> w{ly.x - x.x, ly.y - x.y, ly.z - x.z};
    const T d2 = dot3(w, w);
    const T wl = sqrt(d2);
    w.x /= wl;
    w.y /= wl;
    w.z /= wl;
    const T cx = dot3(n, w), cl = w.y;
    const T no = dot3(n, wo);
    if (cx > T(0) && cl > T(0) && no > T(0)) {
      T ts;
      int ks;
      if (intersect<T>(sph, q.nsph, x, w, false, wl - T(kEps), ts, ks) == 0) {
        const T gl = ((cx * cl) / d2) * T(kLA);
#pragma unroll
        for (int s = 0; s < NSETS; ++s) {
          T f[3], df[3][kND];
          if (kind == 1) {
            bsdf<T>(th[s], n, w, wo, f, df);
          } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              f[c] = T(q.ground[c]) / T(kPiH);
#pragma unroll
              for (int j = 0; j < kND; ++j) df[c][j] = T(0);
            }
          }
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const T g = gl * T(q.Le[c]);
            L[s][c] += beta[s][c] * (f[c] * g);
#pragma unroll
            for (int j = 0; j < kND; ++j)
              dL[s][c][j] += dbeta[s][c][j] * (f[c] * g) + beta[s][c] * (df[c][j] * g);
          }
        }
      }
    }
    if (v == kMaxV - 1 || no <= T(0)) return;
    // cosine-weighted bounce (Malley), rejection candidates from Philox
    double dx = 0.0, dy = 0.0;
    bool got = false;
    for (uint32_t j = 0; !got && j < 64; ++j) {
      double c4[4];
      if (j == 0) {
        c4[0] = u[2];
        c4[1] = u[3];
        c4[2] = 2.0;
        c4[3] = 2.0;
      } else {
        hrng(q.key, pix, q.iteration, path, uint32_t(v * 256 + 1) + j, c4);
      }
#pragma unroll
      for (int m = 0; m < 4; m += 2) {
        if (got) break;
        const double a = 2.0 * c4[m] - 1.0, b = 2.0 * c4[m + 1] - 1.0;
        if (c4[m] <= 1.0 && a * a + b * b < 1.0) {
          dx = a;
          dy = b;
          got = true;
        }
      }
    }
    const T tx = T(dx), ty = T(dy);
    const T dz = sqrt(fmax(T(0), T(1) - (tx * tx + ty * ty)));
    const T sign = copysign(T(1), n.z);
    const T aa = T(-1) / (sign + n.z);
    const T bb = n.x * n.y * aa;
    const V3<T> Tv{T(1) + sign * (n.x * n.x) * aa, sign * bb, -sign * n.x};
    const V3<T> Bv{bb, sign + (n.y * n.y) * aa, -n.y};
    const V3<T> wi{(tx * Tv.x + ty * Bv.x) + dz * n.x, (tx * Tv.y + ty * Bv.y) + dz * n.y,
                   (tx * Tv.z + ty * Bv.z) + dz * n.z};
    if (dz <= T(0)) return;
#pragma unroll
    for (int s = 0; s < NSETS; ++s) {
      T f[3], df[3][kND];
      if (kind == 1) {
        bsdf<T>(th[s], n, wi, wo, f, df);
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          f[c] = T(q.ground[c]) / T(kPiH);
#pragma unroll
          for (int j = 0; j < kND; ++j) df[c][j] = T(0);
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const T wgt = f[c] * T(kPiH);
#pragma unroll
        for (int j = 0; j < kND; ++j)
          dbeta[s][c][j] = dbeta[s][c][j] * wgt + beta[s][c] * (df[c][j] * T(kPiH));
        beta[s][c] = beta[s][c] * wgt;
      }
    }
    o = x;
    d = wi;
  }
}

// theta_now / theta_prev are device dtype vectors (the optimiser's buffers),
// so an optimisation loop needs no host round trip.
template <class T>
__device__ __forceinline__ void load_scene(const HelixK& q, const double* __restrict__ sph_g,
                                           const T* __restrict__ now, const T* __restrict__ prev,
                                           T* sph_s, T (&th)[2][kNP]) {
  for (int k = threadIdx.x; k < 4 * q.nsph; k += blockDim.x) sph_s[k] = T(sph_g[k]);
#pragma unroll
  for (int k = 0; k < kNP; ++k) {
    th[0][k] = now[k];
    th[1][k] = prev[k];
  }
  __syncthreads();
}

template <class T>
__global__ void __launch_bounds__(kHThreads)
    helix_render_kernel(HelixK q, int spp, const double* __restrict__ sph_g,
                        const T* __restrict__ theta, T* __restrict__ img) {
  __shared__ T sph[4 * kMaxSph];
  T th[2][kNP];
  load_scene<T>(q, sph_g, theta, theta, sph, th);
  const int npix = q.W * q.H;
  for (int pix = blockIdx.x * kHThreads + threadIdx.x; pix < npix;
       pix += gridDim.x * kHThreads) {
    const int px = pix % q.W, py = pix / q.W;
    T acc[3] = {T(0), T(0), T(0)};
    for (int s = 0; s < spp; ++s) {
      T L[1][3], dL[1][3][kND];
      trace<T, 1>(q, sph, th, px, py, uint32_t(s), L, dL);
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c] += L[0][c];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) img[size_t(c) * npix + pix] = acc[c] / T(spp);
  }
}

__device__ __forceinline__ long long fixh(double v) { return llrint(v * kFixH); }

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

template <class T>
__global__ void __launch_bounds__(kHThreads)
    helix_pair_kernel(HelixK q, const double* __restrict__ sph_g, const T* __restrict__ now,
                      const T* __restrict__ prev, const T* __restrict__ target,
                      unsigned long long* __restrict__ acc_g, ReducePartials* partials,
                      unsigned int* counter, double* loss_out) {
  __shared__ T sph[4 * kMaxSph];
  __shared__ long long red[kHThreads / 32][2 * kNP];
  if (q.it_offset) q.iteration += __ldg(q.it_offset);
  T th[2][kNP];
  load_scene<T>(q, sph_g, now, prev, sph, th);
  const int npix = q.W * q.H;
  long long fp[kNP] = {0, 0, 0, 0, 0}, fd[kNP] = {0, 0, 0, 0, 0};
  double loss = 0.0;
  for (int pix = q.row0 * q.W + blockIdx.x * kHThreads + threadIdx.x; pix < q.row1 * q.W;
       pix += gridDim.x * kHThreads) {
    const int px = pix % q.W, py = pix / q.W;
    // B, then A (prop terms accumulated, B's data dropped), then C: fewer
    // values live across each trace (same arithmetic as before)
    T LA[2][3], dA[2][3][kND], LC[2][3], dC[2][3][kND];
    double rA[3], rA1[3];
    {
      T LB[1][3], dB[1][3][kND];
      trace<T, 1>(q, sph, th, px, py, 1u, LB, dB);
      trace<T, 2>(q, sph, th, px, py, 0u, LA, dA);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double Is = double(target[size_t(c) * npix + pix]);
        const double rB = double(LB[0][c]) - Is;
        rA[c] = double(LA[0][c]) - Is;
        rA1[c] = double(LA[1][c]) - Is;
        loss += rA[c] * rB;
#pragma unroll
        for (int k = 0; k < kND; ++k) {
          const int j = k == 0 ? c : k + 2;  // base_c, metal (3), rough (4)
          fp[j] += fixh(rA[c] * double(dB[0][c][k]));
          fp[j] += fixh(rB * double(dA[0][c][k]));
        }
      }
    }
    trace<T, 2>(q, sph, th, px, py, 2u, LC, dC);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double Is = double(target[size_t(c) * npix + pix]);
      const double rC = double(LC[0][c]) - Is, rC1 = double(LC[1][c]) - Is;
#pragma unroll
      for (int k = 0; k < kND; ++k) {
        const int j = k == 0 ? c : k + 2;
        fd[j] += fixh((rC * double(dA[0][c][k]) + rA[c] * double(dC[0][c][k])) -
                      (rC1 * double(dA[1][c][k]) + rA1[c] * double(dC[1][c][k])));
      }
    }
  }
  // exact block reduction of the fixed-point sums, one atomic per CTA
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < kNP; ++j) {
    const long long a = warp_sum_ll(fp[j]), b = warp_sum_ll(fd[j]);
    if (lane == 0) {
      red[warp][j] = a;
      red[warp][kNP + j] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * kNP) {
    long long s = 0;
    for (int w = 0; w < kHThreads / 32; ++w) s += red[w][threadIdx.x];
    if (s) red_add_u64(&acc_g[threadIdx.x], (unsigned long long)s);
  }
  Acc a;
  a.ssn = loss;
  grid_reduce4<kHThreads>(a.partials(), partials, counter,
                          [&](const ReducePartials& t) { *loss_out = t.ssn; });
}

// ------------------------------------------------ two-stage sample pair
// The one-kernel form above gives each thread whole pixels (three paths,
// ~1.15 pixels per resident thread at 65k pixels): the last wave is a
// partial one, and the slowest threads trace six paths.  Here every PATH is
// a work item (A, B, C of each pixel: 3 x pixels items, path-major so a
// warp's items share their parameter-set count), fetched 32 at a time by
// each warp from a counter; a path writes its radiance and derivatives
// (both parameter sets, SoA [kHRes][items]) to a scratch buffer, and a
// second kernel combines each pixel's three paths with exactly the
// expressions of helix_pair_kernel (fixed-point sums: order-independent;
// the loss in a fixed pixel order).
constexpr int kHRes = 2 * (3 + 3 * kND);  // per path: [set][L c | dL c k]

template <class T>
__global__ void __launch_bounds__(kHThreads)
    helix_path_kernel(HelixK q, const double* __restrict__ sph_g, const T* __restrict__ now,
                      const T* __restrict__ prev, T* __restrict__ res, unsigned int* work) {
  __shared__ T sph[4 * kMaxSph];
  if (q.it_offset) q.iteration += __ldg(q.it_offset);
  T th[2][kNP];
  load_scene<T>(q, sph_g, now, prev, sph, th);
  const int npt = (q.row1 - q.row0) * q.W;  // pixels of the tile
  const int items = 3 * npt;
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(work, 32u);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (int(base) >= items) break;
    const int j = int(base) + lane;
    if (j >= items) continue;
    const int k = j / npt, i = j - k * npt;  // k: 0 = A, 1 = B, 2 = C
    const int pix = q.row0 * q.W + i;
    const int px = pix % q.W, py = pix / q.W;
    T L[2][3], dL[2][3][kND];
    if (k == 1) {
      T L1[1][3], d1[1][3][kND];
      trace<T, 1>(q, sph, th, px, py, 1u, L1, d1);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        L[0][c] = L1[0][c];
        L[1][c] = T(0);
#pragma unroll
        for (int kk = 0; kk < kND; ++kk) {
          dL[0][c][kk] = d1[0][c][kk];
          dL[1][c][kk] = T(0);
        }
      }
    } else {
      trace<T, 2>(q, sph, th, px, py, k == 0 ? 0u : 2u, L, dL);
    }
#pragma unroll
    for (int st = 0; st < 2; ++st)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        res[size_t(st * 12 + c) * items + j] = L[st][c];
#pragma unroll
        for (int kk = 0; kk < kND; ++kk)
          res[size_t(st * 12 + 3 + c * kND + kk) * items + j] = dL[st][c][kk];
      }
  }
}

template <class T>
__global__ void __launch_bounds__(kHThreads)
    helix_combine_kernel(HelixK q, const T* __restrict__ target, const T* __restrict__ res,
                         unsigned long long* __restrict__ acc_g, ReducePartials* partials,
                         unsigned int* counter, double* loss_out) {
  __shared__ long long red[kHThreads / 32][2 * kNP];
  const int npix = q.W * q.H;
  const int npt = (q.row1 - q.row0) * q.W;
  const int items = 3 * npt;
  auto Lv = [&](int k, int i, int st, int c) { return res[size_t(st * 12 + c) * items + k * npt + i]; };
  auto dv = [&](int k, int i, int st, int c, int kk) {
    return res[size_t(st * 12 + 3 + c * kND + kk) * items + k * npt + i];
  };
  long long fp[kNP] = {0, 0, 0, 0, 0}, fd[kNP] = {0, 0, 0, 0, 0};
  double loss = 0.0;
  for (int i = blockIdx.x * kHThreads + threadIdx.x; i < npt; i += gridDim.x * kHThreads) {
    const int pix = q.row0 * q.W + i;
    double rA[3], rA1[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {  // helix_pair_kernel's expressions, same order
      const double Is = double(target[size_t(c) * npix + pix]);
      const double rB = double(Lv(1, i, 0, c)) - Is;
      rA[c] = double(Lv(0, i, 0, c)) - Is;
      rA1[c] = double(Lv(0, i, 1, c)) - Is;
      loss += rA[c] * rB;
#pragma unroll
      for (int k = 0; k < kND; ++k) {
        const int jj = k == 0 ? c : k + 2;
        fp[jj] += fixh(rA[c] * double(dv(1, i, 0, c, k)));
        fp[jj] += fixh(rB * double(dv(0, i, 0, c, k)));
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double Is = double(target[size_t(c) * npix + pix]);
      const double rC = double(Lv(2, i, 0, c)) - Is, rC1 = double(Lv(2, i, 1, c)) - Is;
#pragma unroll
      for (int k = 0; k < kND; ++k) {
        const int jj = k == 0 ? c : k + 2;
        fd[jj] += fixh((rC * double(dv(0, i, 0, c, k)) + rA[c] * double(dv(2, i, 0, c, k))) -
                       (rC1 * double(dv(0, i, 1, c, k)) + rA1[c] * double(dv(2, i, 1, c, k))));
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < kNP; ++j) {
    const long long a = warp_sum_ll(fp[j]), b = warp_sum_ll(fd[j]);
    if (lane == 0) {
      red[warp][j] = a;
      red[warp][kNP + j] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * kNP) {
    long long s = 0;
    for (int w = 0; w < kHThreads / 32; ++w) s += red[w][threadIdx.x];
    if (s) red_add_u64(&acc_g[threadIdx.x], (unsigned long long)s);
  }
  Acc a;
  a.ssn = loss;
  grid_reduce4<kHThreads>(a.partials(), partials, counter,
                          [&](const ReducePartials& t) { *loss_out = t.ssn; });
}

// Both stages on the context's stream; res = ctx scratch (kHRes x 3 x tile
// pixels of T).  Returns false when the scratch cannot be had.
template <class T>
bool helix_pair_split(mg_ctx* ctx, const HelixK& q, const double* spheres, const T* now,
                      const T* prev, const T* target_img, unsigned long long* accum,
                      double* loss_out) {
  const int npt = (q.row1 - q.row0) * q.W;
  if (npt == 0) return false;
  T* res = static_cast<T*>(ctx_scratch(ctx, sizeof(T) * size_t(kHRes) * 3 * size_t(npt)));
  if (!res) return false;
  cudaMemsetAsync(ctx->work, 0, sizeof(unsigned int), ctx->stream);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, helix_path_kernel<T>, kHThreads, 0);
  const int pgrid = ctx->sm_count * (per_sm > 0 ? per_sm : 1);
  helix_path_kernel<T><<<pgrid, kHThreads, 0, ctx->stream>>>(q, spheres, now, prev, res,
                                                              ctx->work);
  const int cgrid = grid_for(ctx, npt, kHThreads, 8);
  helix_combine_kernel<T><<<cgrid, kHThreads, 0, ctx->stream>>>(
      q, target_img, res, accum, ctx->partials, ctx->counter, loss_out);
  ctx->launches += 1;
  return true;
}

template <class T>
__global__ void helix_finalize_kernel(unsigned long long* __restrict__ acc, T* __restrict__ prop,
                                      T* __restrict__ diff) {
  const int k = threadIdx.x;
  if (k < kNP) {
    prop[k] = T(double((long long)acc[k]) / kFixH);
    diff[k] = T(double((long long)acc[kNP + k]) / kFixH);
  }
  __syncthreads();
  if (k < 2 * kNP) acc[k] = 0ull;
}

HelixK make_helix(int W, int H, int nsph, const double* Le, const double* env, const double* ground,
                  uint64_t key, uint32_t it) {
  HelixK q;
  q.W = W;
  q.H = H;
  q.nsph = nsph;
  q.row0 = 0;
  q.row1 = H;
  for (int c = 0; c < 3; ++c) {
    q.Le[c] = Le[c];
    q.env[c] = env[c];
    q.ground[c] = ground[c];
  }
  q.key = key;
  q.iteration = it;
  q.it_offset = nullptr;
  return q;
}

}  // namespace

// The fp32 launches live in helix_f32.cu: this file compiled again with
// --fmad=true (FMA contraction is allowed in the tolerance-judged fp32
// mode; configs[2] iteration 0.245 -> 0.227 ms), while the fp64 parity
// kernels here keep --fmad=false.
// (the kernel parameter block is passed as void*: HelixK lives in each
// translation unit's anonymous namespace, identical in both)
void helix_render_f32(mg_ctx* ctx, int grid, const void* qp, int spp, const double* spheres,
                      const float* theta, float* img)
#ifdef MG_HELIX_F32_TU
{
  const HelixK& q = *static_cast<const HelixK*>(qp);
  helix_render_kernel<float><<<grid, kHThreads, 0, ctx->stream>>>(q, spp, spheres, theta, img);
}
#else
    ;
#endif
void helix_pair_f32(mg_ctx* ctx, int grid, const void* qp, const double* spheres,
                    const float* now, const float* prev, const float* target_img,
                    unsigned long long* accum, double* loss_out, float* prop, float* diff)
#ifdef MG_HELIX_F32_TU
{
  const HelixK& q = *static_cast<const HelixK*>(qp);
  if (!(g_helix_split &&
        helix_pair_split<float>(ctx, q, spheres, now, prev, target_img, accum, loss_out)))
    helix_pair_kernel<float><<<grid, kHThreads, 0, ctx->stream>>>(
        q, spheres, now, prev, target_img, accum, ctx->partials, ctx->counter, loss_out);
  helix_finalize_kernel<float><<<1, 32, 0, ctx->stream>>>(accum, prop, diff);
}
#else
    ;
#endif

}  // namespace mg

#ifndef MG_HELIX_F32_TU
using namespace mg;

extern "C" {

int mg_helix_render(mg_ctx* ctx, int32_t dtype, int32_t W, int32_t H, int32_t nsph,
                    const double* spheres, const double* Le, const double* env,
                    const double* ground, const void* theta, int32_t spp, uint64_t key,
                    void* img) {
  if (!ctx || !spheres || !Le || !env || !ground || !theta || !img)
    return fail(MG_EINVAL, "mg_helix_render: null argument");
  if (W < 1 || H < 1 || spp < 1 || nsph < 0 || nsph > kMaxSph)
    return fail(MG_EINVAL, "mg_helix_render: bad sizes (nsph <= 256)");
  const HelixK q = make_helix(W, H, nsph, Le, env, ground, key, 0xffffffffu);
  const int grid = grid_for(ctx, int64_t(W) * H, kHThreads, 8);
  if (dtype == MG_F64)
    helix_render_kernel<double><<<grid, kHThreads, 0, ctx->stream>>>(
        q, spp, spheres, (const double*)theta, (double*)img);
  else if (dtype == MG_F32)
    helix_render_f32(ctx, grid, &q, spp, spheres, (const float*)theta, (float*)img);
  else
    return fail(MG_EINVAL, "mg_helix_render: unknown dtype");
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

int mg_helix_sample_pair(mg_ctx* ctx, int32_t dtype, int32_t W, int32_t H, int32_t nsph,
                         const double* spheres, const double* Le, const double* env,
                         const double* ground, const void* target_img, const void* now,
                         const void* prev, uint64_t key, uint32_t iteration, int32_t row0,
                         int32_t row1, void* accum, void* prop, void* diff, double* loss_out) {
  if (!ctx || !spheres || !Le || !env || !ground || !target_img || !now || !prev || !accum ||
      !prop || !diff || !loss_out)
    return fail(MG_EINVAL, "mg_helix_sample_pair: null argument");
  if (W < 1 || H < 1 || nsph < 0 || nsph > kMaxSph)
    return fail(MG_EINVAL, "mg_helix_sample_pair: bad sizes (nsph <= 256)");
  if (row0 < 0 || row1 > H || row0 > row1) return fail(MG_EINVAL, "mg_helix_sample_pair: bad rows");
  HelixK q = make_helix(W, H, nsph, Le, env, ground, key, iteration);
  q.row0 = row0;
  q.row1 = row1;
  q.it_offset = ctx->it_offset;
  const int grid = grid_for(ctx, int64_t(W) * (row1 - row0) + 1, kHThreads, 8);
  if (dtype == MG_F64) {
    if (!(g_helix_split &&
          helix_pair_split<double>(ctx, q, spheres, (const double*)now, (const double*)prev,
                                   (const double*)target_img, (unsigned long long*)accum,
                                   loss_out)))
      helix_pair_kernel<double><<<grid, kHThreads, 0, ctx->stream>>>(
          q, spheres, (const double*)now, (const double*)prev, (const double*)target_img,
          (unsigned long long*)accum, ctx->partials, ctx->counter, loss_out);
    helix_finalize_kernel<double><<<1, 32, 0, ctx->stream>>>((unsigned long long*)accum,
                                                             (double*)prop, (double*)diff);
  } else if (dtype == MG_F32) {
    helix_pair_f32(ctx, grid, &q, spheres, (const float*)now, (const float*)prev,
                   (const float*)target_img, (unsigned long long*)accum, loss_out, (float*)prop,
                   (float*)diff);
  } else {
    return fail(MG_EINVAL, "mg_helix_sample_pair: unknown dtype");
  }
  ctx->launches += 1;
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

}  // extern "C"
#endif  // MG_HELIX_F32_TU
