// F1 slice 3 (BASELINE.json configs[3]): gradient samples for texture
// optimisation on a triangle-mesh scene — quad, tessellated sphere and a
// seeded displaced-sphere mesh, each with its own R x R RGB albedo +
// roughness texture — path traced to depth 6 with next-event estimation.
// Scene, estimators and the CPU oracle: DESIGN.md §12 and
// oracle/metagrad_oracle.c mgo_mesh_* (the reference has no renderer).
//
// * BVH: binned-SAH build on the host, nodes relabelled breadth-first so
//   the top levels are one contiguous block that every CTA stages in shared
//   memory; boxes are fp32, rounded outwards and padded, so the fp32 slab
//   test never culls a triangle the fp64 Moller-Trumbore test would hit —
//   the closest hit (ties -> lower original triangle index) equals the
//   oracle's brute-force answer bit for bit.
// * One thread per pixel traces paths A (both parameter sets: shared
//   geometry, two BSDF evaluations), B and C; sampling is independent of
//   the parameters.  Path A's per-vertex adjoint data is stored, suffix
//   radiance accumulated backwards, and every (vertex, parameter)
//   contribution is added as a 2^-40 fixed-point int64 atomic into the
//   texture's prop / diff accumulators (order independent, deterministic).
//   Path B is traced twice (radiance first, then with storage) so that only
//   one path's vertex data is live at a time.
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <vector>

#include "mg_common.cuh"
#include "philox.cuh"

struct mg_mesh_scene {
  int T = 0, nobj = 0, R = 0, nnodes = 0, depth = 0, nch = 4;
  double* tri = nullptr;   // [T][18] in BVH order
  int* orig = nullptr;     // [T] original triangle index
  int* obj = nullptr;      // [T] object id (BVH order)
  float4* nodes = nullptr; // [2 * nnodes]: (lo.xyz, a) (hi.xyz, b)
  unsigned int* work = nullptr;  // pixel work counter of the pair kernel
  void* wf = nullptr;            // wavefront path state (grow-only)
  size_t wf_cap = 0;
};

namespace mg {
// mg_set_option("mesh_megakernel", 1): one-thread-per-pixel megakernel
// instead of the default wavefront stages (A/B comparison; identical results)
bool g_mesh_megakernel = false;
// mg_set_option("bvh_leaf_size", k): maximum triangles per BVH leaf (1..7),
// applied to scenes created afterwards
int g_bvh_leaf = 2;
namespace {

constexpr int kMThreads = 128;
constexpr int kMaxV = 8;
constexpr int kRec = 18;
constexpr int kSmemNodes = 256;  // top BVH levels staged in shared memory (16 KB)
constexpr int kStackDepth = 48;  // traversal stack per thread, in shared memory
constexpr double kTMin = 1e-9, kOff = 1e-6;
constexpr double kPiM = 3.14159265358979323846;
constexpr double kFixM = 1099511627776.0;  // 2^40

// ------------------------------------------------------------ host BVH
struct TmpNode {
  double lo[3], hi[3];
  int left = -1, right = -1, first = 0, count = 0;
};

struct Builder {
  const double* tri;
  std::vector<double> blo, bhi, cen;  // [T][3]
  std::vector<int> idx;
  std::vector<TmpNode> nodes;
  int max_depth = 0;
  bool too_deep = false;

  void bounds(int b, int e, double lo[3], double hi[3], bool centroids) const {
    for (int k = 0; k < 3; ++k) {
      lo[k] = INFINITY;
      hi[k] = -INFINITY;
    }
    for (int i = b; i < e; ++i) {
      const int t = idx[size_t(i)];
      for (int k = 0; k < 3; ++k) {
        const double l = centroids ? cen[size_t(3 * t + k)] : blo[size_t(3 * t + k)];
        const double h = centroids ? cen[size_t(3 * t + k)] : bhi[size_t(3 * t + k)];
        lo[k] = std::min(lo[k], l);
        hi[k] = std::max(hi[k], h);
      }
    }
  }
  static double area(const double lo[3], const double hi[3]) {
    const double x = hi[0] - lo[0], y = hi[1] - lo[1], z = hi[2] - lo[2];
    return (x < 0 || y < 0 || z < 0) ? 0.0 : 2.0 * (x * y + y * z + z * x);
  }

  int build(int b, int e, int depth) {
    max_depth = std::max(max_depth, depth);
    const int id = int(nodes.size());
    nodes.emplace_back();
    TmpNode nd;
    bounds(b, e, nd.lo, nd.hi, false);
    const int n = e - b;
    auto make_leaf = [&]() {
      nd.first = b;
      nd.count = n;
      nodes[size_t(id)] = nd;
      return id;
    };
    if (n <= g_bvh_leaf) return make_leaf();
    if (depth >= kStackDepth - 2) {  // deeper than the traversal stack allows
      too_deep = true;
      return make_leaf();
    }
    double clo[3], chi[3];
    bounds(b, e, clo, chi, true);
    int axis = 0;
    for (int k = 1; k < 3; ++k)
      if (chi[k] - clo[k] > chi[axis] - clo[axis]) axis = k;
    const double ext = chi[axis] - clo[axis];
    int mid = -1;
    if (ext > 0.0) {
      constexpr int kBins = 16;
      int cnt[kBins] = {0};
      double bl[kBins][3], bh[kBins][3];
      for (int i = 0; i < kBins; ++i)
        for (int k = 0; k < 3; ++k) {
          bl[i][k] = INFINITY;
          bh[i][k] = -INFINITY;
        }
      auto bin_of = [&](int t) {
        int q = int(((cen[size_t(3 * t + axis)] - clo[axis]) / ext) * kBins);
        return q < 0 ? 0 : (q >= kBins ? kBins - 1 : q);
      };
      for (int i = b; i < e; ++i) {
        const int t = idx[size_t(i)], q = bin_of(t);
        cnt[q]++;
        for (int k = 0; k < 3; ++k) {
          bl[q][k] = std::min(bl[q][k], blo[size_t(3 * t + k)]);
          bh[q][k] = std::max(bh[q][k], bhi[size_t(3 * t + k)]);
        }
      }
      double best = INFINITY;
      int best_split = -1;
      for (int s = 1; s < kBins; ++s) {
        double l0[3] = {INFINITY, INFINITY, INFINITY}, h0[3] = {-INFINITY, -INFINITY, -INFINITY};
        double l1[3] = {INFINITY, INFINITY, INFINITY}, h1[3] = {-INFINITY, -INFINITY, -INFINITY};
        int n0 = 0, n1 = 0;
        for (int q = 0; q < kBins; ++q) {
          double* L = q < s ? l0 : l1;
          double* H = q < s ? h0 : h1;
          (q < s ? n0 : n1) += cnt[q];
          for (int k = 0; k < 3; ++k) {
            L[k] = std::min(L[k], bl[q][k]);
            H[k] = std::max(H[k], bh[q][k]);
          }
        }
        if (!n0 || !n1) continue;
        const double c = area(l0, h0) * n0 + area(l1, h1) * n1;
        if (c < best) {
          best = c;
          best_split = s;
        }
      }
      if (best_split > 0) {
        auto it = std::partition(idx.begin() + b, idx.begin() + e,
                                 [&](int t) { return bin_of(t) < best_split; });
        mid = int(it - idx.begin());
      }
    }
    if (mid <= b || mid >= e) {  // degenerate: median split on the axis
      mid = (b + e) / 2;
      std::nth_element(idx.begin() + b, idx.begin() + mid, idx.begin() + e, [&](int x, int y) {
        const double cx = cen[size_t(3 * x + axis)], cy = cen[size_t(3 * y + axis)];
        return cx < cy || (cx == cy && x < y);
      });
    }
    const int l = build(b, mid, depth + 1);
    const int r = build(mid, e, depth + 1);
    nd.left = l;
    nd.right = r;
    nodes[size_t(id)] = nd;
    return id;
  }
};

// ------------------------------------------------------------ device
struct MeshDev {
  const double* __restrict__ tri;
  const int* __restrict__ orig;
  const int* __restrict__ obj;
  const float4* __restrict__ nodes;
  int nnodes;
};

struct MeshK {
  int W, H, R, nobj, nch;
  int row0, row1;
  double view[25];
  uint64_t key;
  uint32_t iteration;
};

__device__ __forceinline__ double dot3d(const double a[3], const double b[3]) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

__device__ __forceinline__ void cross3d(const double a[3], const double b[3], double r[3]) {
  r[0] = a[1] * b[2] - a[2] * b[1];
  r[1] = a[2] * b[0] - a[0] * b[2];
  r[2] = a[0] * b[1] - a[1] * b[0];
}

// Moller-Trumbore in fp64, same operation order as the oracle (ms_tri_hit)
__device__ __forceinline__ bool tri_hit(const double* __restrict__ r, const double o[3],
                                        const double d[3], double& t, double& u, double& v) {
  const double v0[3] = {r[0], r[1], r[2]}, e1[3] = {r[3], r[4], r[5]}, e2[3] = {r[6], r[7], r[8]};
  double p[3], q[3], s[3];
  cross3d(d, e2, p);
  const double det = dot3d(e1, p);
  if (det == 0.0) return false;
  const double inv = 1.0 / det;
  s[0] = o[0] - v0[0];
  s[1] = o[1] - v0[1];
  s[2] = o[2] - v0[2];
  const double uu = dot3d(s, p) * inv;
  if (uu < 0.0 || uu > 1.0) return false;
  cross3d(s, e1, q);
  const double vv = dot3d(d, q) * inv;
  if (vv < 0.0 || uu + vv > 1.0) return false;
  const double tt = dot3d(e2, q) * inv;
  if (!(tt > kTMin)) return false;
  t = tt;
  u = uu;
  v = vv;
  return true;
}

// BVH2 node = the boxes of its two children (64 B, four float4):
//   n0 = c0.lo.xyz c0.hi.x   n1 = c0.hi.yz c1.lo.xy   n2 = c1.lo.z c1.hi.xyz
//   n3 = (ref0, ref1) as int bits; ref >= 0: internal node, ref < 0: leaf
//   with triangles [first, first + count), ~ref = first * 8 + count.
// One 64-byte fetch per traversal step tests both children.
struct Node4 {
  float4 a, b, c, d;
};

__device__ __forceinline__ Node4 load_node(const MeshDev& m, const float4* sn, int i) {
  Node4 n;
  if (i < kSmemNodes) {
    n.a = sn[4 * i];
    n.b = sn[4 * i + 1];
    n.c = sn[4 * i + 2];
    n.d = sn[4 * i + 3];
  } else {
    n.a = __ldg(&m.nodes[4 * i]);
    n.b = __ldg(&m.nodes[4 * i + 1]);
    n.c = __ldg(&m.nodes[4 * i + 2]);
    n.d = __ldg(&m.nodes[4 * i + 3]);
  }
  return n;
}

__device__ __forceinline__ bool slab6(float lx, float ly, float lz, float hx, float hy, float hz,
                                      const float o[3], const float inv[3], float tmax,
                                      float& tnear) {
  const float tx0 = (lx - o[0]) * inv[0], tx1 = (hx - o[0]) * inv[0];
  const float ty0 = (ly - o[1]) * inv[1], ty1 = (hy - o[1]) * inv[1];
  const float tz0 = (lz - o[2]) * inv[2], tz1 = (hz - o[2]) * inv[2];
  const float tn = fmaxf(fmaxf(fminf(tx0, tx1), fminf(ty0, ty1)), fmaxf(fminf(tz0, tz1), 0.0f));
  const float tf = fminf(fminf(fmaxf(tx0, tx1), fmaxf(ty0, ty1)), fminf(fmaxf(tz0, tz1), tmax));
  tnear = tn;
  return tn <= tf;
}

// Triangle record fields 0..8 (v0, e1, e2) with 16-byte loads (records are
// 144 B = 9 x 16 B and the array is 256-byte aligned).
__device__ __forceinline__ bool tri_hit_rec(const double* __restrict__ rec, const double o[3],
                                            const double d[3], double& t, double& u, double& v) {
  const double2* r2 = reinterpret_cast<const double2*>(rec);
  const double2 x0 = __ldg(r2), x1 = __ldg(r2 + 1), x2 = __ldg(r2 + 2), x3 = __ldg(r2 + 3);
  const double r[9] = {x0.x, x0.y, x1.x, x1.y, x2.x, x2.y, x3.x, x3.y, __ldg(rec + 8)};
  return tri_hit(r, o, d, t, u, v);
}

// ANY: any hit with t < tmax (shadow rays).  Otherwise the closest hit with
// t < tmax; ties on t resolve to the lower original triangle index, so the
// answer is the oracle's brute-force scan.  Returns the BVH slot or -1.
// (stk: reserved for a shared-memory stack; the local-memory stack measured
// faster — the shared one cut occupancy.)
template <bool ANY>
__device__ __forceinline__ int trace_impl(const MeshDev& m, const float4* sn, const double o[3],
                                          const double d[3], double tmax, double& t_out,
                                          double& u_out, double& v_out) {
  float of[3], inv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    of[k] = float(o[k]);
    const float dk = float(d[k]);
    inv[k] = 1.0f / (fabsf(dk) > 1e-20f ? dk : copysignf(1e-20f, dk));
  }
  int stack[kStackDepth];
  int sp = 0, node = 0;
  double best = tmax, bu = 0.0, bv = 0.0;
  int bslot = -1, bid = INT_MAX;
  float bestf = __double2float_ru(best);
  for (;;) {
    if (node < 0) {  // leaf: triangles [first, first + count)
      const int first = (~node) >> 3, count = (~node) & 7;
      for (int sidx = first; sidx < first + count; ++sidx) {
        double t, u, v;
        if (!tri_hit_rec(m.tri + size_t(kRec) * sidx, o, d, t, u, v) || !(t <= best)) continue;
        if (ANY) {
          if (t < tmax) return sidx;
          continue;
        }
        const int id = __ldg(&m.orig[sidx]);
        if (t < best || id < bid) {
          best = t;
          bu = u;
          bv = v;
          bslot = sidx;
          bid = id;
          bestf = __double2float_ru(best);
        }
      }
    } else {
      const Node4 n = load_node(m, sn, node);
      float t0, t1;
      const bool h0 = slab6(n.a.x, n.a.y, n.a.z, n.a.w, n.b.x, n.b.y, of, inv, bestf, t0);
      const bool h1 = slab6(n.b.z, n.b.w, n.c.x, n.c.y, n.c.z, n.c.w, of, inv, bestf, t1);
      const int r0 = __float_as_int(n.d.x), r1 = __float_as_int(n.d.y);
      if (h0 && h1) {
        const bool first0 = t0 <= t1;
        stack[sp++] = first0 ? r1 : r0;
        node = first0 ? r0 : r1;
        continue;
      }
      if (h0) {
        node = r0;
        continue;
      }
      if (h1) {
        node = r1;
        continue;
      }
    }
    if (sp == 0) break;
    node = stack[--sp];
  }
  t_out = best;
  u_out = bu;
  v_out = bv;
  return bslot;
}

// out-of-line copy for the megakernel (one body shared by all its call
// sites keeps its instruction footprint small); the wavefront kernels
// inline trace_impl at their single call site.
template <bool ANY>
__device__ __noinline__ int trace(const MeshDev& m, const float4* sn, int* stk, const double o[3],
                                  const double d[3], double tmax, double& t_out, double& u_out,
                                  double& v_out) {
  return trace_impl<ANY>(m, sn, o, d, tmax, t_out, u_out, v_out);
}

__device__ __forceinline__ void prng(uint64_t key, uint32_t pix, uint32_t it, uint32_t path,
                                     uint32_t slot, double u[4]) {
  const Philox4 r =
      philox4x32_10(Philox4{{pix, it, path, slot}}, uint32_t(key), uint32_t(key >> 32));
#pragma unroll
  for (int k = 0; k < 4; ++k) u[k] = double(r.x[k]) * 0x1.0p-32;
}

// principled BSDF with metalness 0 (the helix slice's expressions with
// metal = 0): f_c = base_c / pi + DG F, and dS/drough = dDG/drough F
template <class T>
__device__ __forceinline__ void bsdf_m0(const T base[3], T rough, const T n[3], const T wi[3],
                                        const T wo[3], T f[3], T& dS) {
  const T alpha = T(0.05) + T(0.95) * (rough * rough);
  const T a2 = alpha * alpha;
  T h[3] = {wi[0] + wo[0], wi[1] + wo[1], wi[2] + wo[2]};
  const T hl = sqrt((h[0] * h[0] + h[1] * h[1]) + h[2] * h[2]);
  h[0] /= hl;
  h[1] /= hl;
  h[2] /= hl;
  auto dt = [](const T* a, const T* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; };
  const T nh = dt(n, h), ni = dt(n, wi), no = dt(n, wo), ih = dt(wi, h);
  const T den = nh * nh * (a2 - T(1)) + T(1);
  const T D = a2 / (T(kPiM) * (den * den));
  const T dD_da2 = (den - T(2) * a2 * (nh * nh)) / (T(kPiM) * ((den * den) * den));
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
  const T F0 = T(0.04);
  const T F = F0 + (T(1) - F0) * q5;
#pragma unroll
  for (int c = 0; c < 3; ++c) f[c] = base[c] / T(kPiM) + DG * F;
  dS = dDG_drough * F;
}

// full principled BSDF (configs[4], metalness texture): f[c] and
// df[c][k] = d f_c / d(base_c, metal, rough) — the oracle's hx_bsdf
template <class T>
__device__ __forceinline__ void bsdf_full(const T base[3], T metal, T rough, const T n[3],
                                          const T wi[3], const T wo[3], T f[3], T df[3][3]) {
  const T alpha = T(0.05) + T(0.95) * (rough * rough);
  const T a2 = alpha * alpha;
  T h[3] = {wi[0] + wo[0], wi[1] + wo[1], wi[2] + wo[2]};
  const T hl = sqrt((h[0] * h[0] + h[1] * h[1]) + h[2] * h[2]);
  h[0] /= hl;
  h[1] /= hl;
  h[2] /= hl;
  auto dt = [](const T* a, const T* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; };
  const T nh = dt(n, h), ni = dt(n, wi), no = dt(n, wo), ih = dt(wi, h);
  const T den = nh * nh * (a2 - T(1)) + T(1);
  const T D = a2 / (T(kPiM) * (den * den));
  const T dD_da2 = (den - T(2) * a2 * (nh * nh)) / (T(kPiM) * ((den * den) * den));
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
    const T F0 = T(0.04) * (T(1) - metal) + base[c] * metal;
    const T F = F0 + (T(1) - F0) * q5;
    f[c] = ((T(1) - metal) * base[c]) / T(kPiM) + DG * F;
    df[c][0] = (T(1) - metal) / T(kPiM) + DG * (metal * (T(1) - q5));
    df[c][1] = (-base[c]) / T(kPiM) + DG * ((base[c] - T(0.04)) * (T(1) - q5));
    df[c][2] = dDG_drough * F;
  }
}

template <class T, int NS>
struct PathStore {
  int base[kMaxV];
  T A[NS][kMaxV][3];
  T dSn[NS][kMaxV];
  T invfb[NS][kMaxV][3];
  T dSb[NS][kMaxV];
  T C[NS][kMaxV][3];
};

struct NoStore {};

// One path for NS parameter sets (th[0] = theta_t, th[1] = theta_{t-1});
// radiance L[s][c], environment after the last vertex E[s][c]; per-vertex
// adjoint data into *st when STORE.  Returns the number of vertices.
template <class T, int NS, bool STORE, class Store, int NCH = 4>
__device__ __noinline__ int mesh_path(const MeshK& q, const MeshDev& m, const float4* sn, int* stk,
                                     const T* const th[2],
                         int px, int py, uint32_t it, uint32_t path, T L[NS][3], T E[NS][3],
                         Store* st) {
  const double* V = q.view;
  const int maxv = int(V[24]);
  const int R2 = q.R * q.R;
  const uint32_t pix = uint32_t(py * q.W + px);
  double u[4];
  prng(q.key, pix, it, path, 0u, u);
  const double sx = ((double(px) + u[0]) / double(q.W)) * 2.0 - 1.0;
  const double sy = 1.0 - ((double(py) + u[1]) / double(q.H)) * 2.0;
  const double ax = sx * (V[12] * (double(q.W) / double(q.H))), ay = sy * V[12];
  double o[3] = {V[0], V[1], V[2]};
  double d[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) d[i] = (V[3 + i] + ax * V[6 + i]) + ay * V[9 + i];
  const double dl = sqrt(dot3d(d, d));
  d[0] /= dl;
  d[1] /= dl;
  d[2] /= dl;
  T beta[NS][3];
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      beta[s][c] = T(1);
      L[s][c] = T(0);
      E[s][c] = T(0);
    }
  const double la = (V[15] - V[14]) * (V[17] - V[16]);
  int nv = 0;
  for (int v = 0; v < maxv && v < kMaxV; ++v) {
    double t = INFINITY, bu, bv;
    const int slot = trace<false>(m, sn, stk, o, d, INFINITY, t, bu, bv);
    if (slot < 0) {
#pragma unroll
      for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          E[s][c] = beta[s][c] * T(V[21 + c]);
          L[s][c] += E[s][c];
        }
      return nv;
    }
    const double* r = m.tri + size_t(kRec) * slot;
    const double x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
    double n[3] = {r[9], r[10], r[11]};
    if (dot3d(n, d) > 0.0) {
      n[0] = -n[0];
      n[1] = -n[1];
      n[2] = -n[2];
    }
    const double U = (r[12] + bu * r[14]) + bv * r[16];
    const double W_ = (r[13] + bu * r[15]) + bv * r[17];
    int tx = int(U * q.R), ty = int(W_ * q.R);
    tx = tx < 0 ? 0 : (tx > q.R - 1 ? q.R - 1 : tx);
    ty = ty < 0 ? 0 : (ty > q.R - 1 ? q.R - 1 : ty);
    static_assert(NCH == 4 || !STORE, "stored paths are the configs[3] form");
    const int pbase = __ldg(&m.obj[slot]) * NCH * R2 + ty * q.R + tx;
    if constexpr (STORE) {
      st->base[nv] = pbase;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        st->dSn[s][nv] = T(0);
        st->dSb[s][nv] = T(0);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          st->A[s][nv][c] = T(0);
          st->invfb[s][nv][c] = T(0);
          st->C[s][nv][c] = T(0);
        }
      }
    }
    const int vi = nv;
    ++nv;
    T base[NS][3], rough[NS], metal[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
#pragma unroll
      for (int c = 0; c < 3; ++c) base[s][c] = th[s][pbase + c * R2];
      rough[s] = th[s][pbase + 3 * R2];
      metal[s] = NCH == 5 ? th[s][pbase + 4 * R2] : T(0);
    }
    const double wo[3] = {-d[0], -d[1], -d[2]};
    const double xo[3] = {x[0] + kOff * n[0], x[1] + kOff * n[1], x[2] + kOff * n[2]};
    prng(q.key, pix, it, path, uint32_t(v * 256 + 1), u);
    const double lp[3] = {V[14] + u[0] * (V[15] - V[14]), V[13], V[16] + u[1] * (V[17] - V[16])};
    double w[3] = {lp[0] - x[0], lp[1] - x[1], lp[2] - x[2]};
    const double d2 = dot3d(w, w);
    const double wl = sqrt(d2);
    w[0] /= wl;
    w[1] /= wl;
    w[2] /= wl;
    const double cx = dot3d(n, w), cl = w[1];
    const T nT[3] = {T(n[0]), T(n[1]), T(n[2])}, woT[3] = {T(wo[0]), T(wo[1]), T(wo[2])};
    if (cx > 0.0 && cl > 0.0 && dot3d(n, wo) > 0.0) {
      double ts, tu, tv;
      if (trace<true>(m, sn, stk, xo, w, wl - kOff, ts, tu, tv) < 0) {
        const double gl = ((cx * cl) / d2) * la;
        const T wT[3] = {T(w[0]), T(w[1]), T(w[2])};
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          T f[3], dS;
          if constexpr (NCH == 5) {
            T df[3][3];
            bsdf_full<T>(base[s], metal[s], rough[s], nT, wT, woT, f, df);
          } else {
            bsdf_m0<T>(base[s], rough[s], nT, wT, woT, f, dS);
          }
          if constexpr (STORE) st->dSn[s][vi] = dS;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const T A = beta[s][c] * T(gl * V[18 + c]);
            const T Cc = A * f[c];
            if constexpr (STORE) {
              st->A[s][vi][c] = A;
              st->C[s][vi][c] = Cc;
            }
            L[s][c] += Cc;
          }
        }
      }
    }
    if (v == maxv - 1 || dot3d(n, wo) <= 0.0) return nv;
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
        prng(q.key, pix, it, path, uint32_t(v * 256 + 1) + j, c4);
      }
#pragma unroll
      for (int mm = 0; mm < 4; mm += 2) {
        if (got) break;
        const double a = 2.0 * c4[mm] - 1.0, b = 2.0 * c4[mm + 1] - 1.0;
        if (c4[mm] <= 1.0 && a * a + b * b < 1.0) {
          dx = a;
          dy = b;
          got = true;
        }
      }
    }
    const double dz = sqrt(fmax(0.0, 1.0 - (dx * dx + dy * dy)));
    if (dz <= 0.0) return nv;
    // Duff et al. orthonormal basis (oracle hx_onb)
    const double sign = copysign(1.0, n[2]);
    const double aa = -1.0 / (sign + n[2]);
    const double bb = n[0] * n[1] * aa;
    const double Tb[3] = {1.0 + sign * (n[0] * n[0]) * aa, sign * bb, -sign * n[0]};
    const double Bb[3] = {bb, sign + (n[1] * n[1]) * aa, -n[1]};
    const double wi[3] = {(dx * Tb[0] + dy * Bb[0]) + dz * n[0],
                          (dx * Tb[1] + dy * Bb[1]) + dz * n[1],
                          (dx * Tb[2] + dy * Bb[2]) + dz * n[2]};
    const T wiT[3] = {T(wi[0]), T(wi[1]), T(wi[2])};
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      T f[3], dS;
      if constexpr (NCH == 5) {
        T df[3][3];
        bsdf_full<T>(base[s], metal[s], rough[s], nT, wiT, woT, f, df);
      } else {
        bsdf_m0<T>(base[s], rough[s], nT, wiT, woT, f, dS);
      }
      if constexpr (STORE) st->dSb[s][vi] = dS;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if constexpr (STORE) st->invfb[s][vi][c] = f[c] != T(0) ? T(1) / f[c] : T(0);
        beta[s][c] = beta[s][c] * (f[c] * T(kPiM));
      }
    }
    o[0] = xo[0];
    o[1] = xo[1];
    o[2] = xo[2];
    d[0] = wi[0];
    d[1] = wi[1];
    d[2] = wi[2];
  }
  return nv;
}

__device__ __forceinline__ unsigned long long fixq(double v) {
  return (unsigned long long)llrint(v * kFixM);
}

// adjoint of a stored path, set s, channel weights w (oracle ms_scatter)
template <class T, int NS>
__device__ __noinline__ void scatter(const PathStore<T, NS>& st, int nv, const T E[3], int s, const T w[3],
                        int R2, unsigned long long* __restrict__ acc) {
  T Q[3] = {E[0], E[1], E[2]};
  for (int v = nv - 1; v >= 0; --v) {
    T gr = T(0);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const T gb = w[c] * ((st.A[s][v][c] / T(kPiM)) + Q[c] * (st.invfb[s][v][c] / T(kPiM)));
      atomicAdd(&acc[st.base[v] + c * R2], fixq(double(gb)));
      gr += w[c] * (st.A[s][v][c] * st.dSn[s][v] + Q[c] * (st.invfb[s][v][c] * st.dSb[s][v]));
    }
    atomicAdd(&acc[st.base[v] + 3 * R2], fixq(double(gr)));
#pragma unroll
    for (int c = 0; c < 3; ++c) Q[c] = Q[c] + st.C[s][v][c];
  }
}

__device__ __forceinline__ void stage_nodes(const MeshDev& m, float4* sn) {
  const int n = 4 * (m.nnodes < kSmemNodes ? m.nnodes : kSmemNodes);
  for (int i = threadIdx.x; i < n; i += blockDim.x) sn[i] = m.nodes[i];
  __syncthreads();
}

// shared-memory arrays every tracing kernel declares
#define MESH_SMEM                       \
  __shared__ float4 sn[4 * kSmemNodes]; \
  int* stk = nullptr;                   \
  stage_nodes(m, sn)

template <class T, int NCH>
__global__ void __launch_bounds__(kMThreads)
    mesh_render_kernel(MeshK q, MeshDev m, int spp, const T* __restrict__ theta,
                       T* __restrict__ img) {
  MESH_SMEM;
  const int npix = q.W * q.H;
  const T* th[2] = {theta, theta};
  for (int pix = blockIdx.x * kMThreads + threadIdx.x; pix < npix; pix += gridDim.x * kMThreads) {
    const int px = pix % q.W, py = pix / q.W;
    double acc[3] = {0.0, 0.0, 0.0};
    for (int s = 0; s < spp; ++s) {
      T L[1][3], E[1][3];
      mesh_path<T, 1, false, NoStore, NCH>(q, m, sn, stk, th, px, py, 0xffffffffu, uint32_t(s),
                                           L, E, nullptr);
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c] += double(L[0][c]);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) img[size_t(c) * npix + pix] = T(acc[c] / double(spp));
  }
}

// Pixels are handed out 32 at a time from a global counter (one atomic
// per warp), so warps that drew short paths take more pixels and the CTAs
// finish together (the path length varies 1..maxv per pixel).
__device__ __forceinline__ int next_pixels(unsigned int* work) {
  int base = 0;
  if ((threadIdx.x & 31) == 0) base = int(atomicAdd(work, 32u));
  return __shfl_sync(0xffffffffu, base, 0);
}

template <class T>
__global__ void __launch_bounds__(kMThreads)
    mesh_pair_kernel(MeshK q, MeshDev m, const T* __restrict__ target_img,
                     const T* __restrict__ now, const T* __restrict__ prev,
                     unsigned long long* __restrict__ acc, long long np, unsigned int* work,
                     ReducePartials* partials, unsigned int* counter, double* loss_out) {
  MESH_SMEM;
  const int npix = q.W * q.H;
  const int R2 = q.R * q.R;
  const T* th[2] = {now, prev};
  const int pix0 = q.row0 * q.W, pix1 = q.row1 * q.W;
  double loss = 0.0;
  for (int wbase = next_pixels(work); pix0 + wbase < pix1; wbase = next_pixels(work)) {
    const int pix = pix0 + wbase + int(threadIdx.x & 31);
    if (pix >= pix1) continue;
    const int px = pix % q.W, py = pix / q.W;
    T LB[1][3], EB[1][3], LC[2][3], EC[2][3], LA[2][3], EA[2][3];
    mesh_path<T, 1, false, NoStore>(q, m, sn, stk, th, px, py, q.iteration, 1u, LB, EB, nullptr);
    mesh_path<T, 2, false, NoStore>(q, m, sn, stk, th, px, py, q.iteration, 2u, LC, EC, nullptr);
    T rA[3], rB[3], wC0[3], wC1[3];
    {
      PathStore<T, 2> st;
      const int na =
          mesh_path<T, 2, true>(q, m, sn, stk, th, px, py, q.iteration, 0u, LA, EA, &st);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const T Is = target_img[size_t(c) * npix + pix];
        rA[c] = LA[0][c] - Is;
        rB[c] = LB[0][c] - Is;
        wC0[c] = T(2) * (LC[0][c] - Is);
        wC1[c] = T(-2) * (LC[1][c] - Is);
        loss += double(rA[c] * rB[c]);
      }
      scatter<T, 2>(st, na, EA[0], 0, rB, R2, acc);
      scatter<T, 2>(st, na, EA[0], 0, wC0, R2, acc + np);
      scatter<T, 2>(st, na, EA[1], 1, wC1, R2, acc + np);
    }
    {
      PathStore<T, 1> st;
      const int nb =
          mesh_path<T, 1, true>(q, m, sn, stk, th, px, py, q.iteration, 1u, LB, EB, &st);
      scatter<T, 1>(st, nb, EB[0], 0, rA, R2, acc);
    }
  }
  Acc a;
  a.ssn = loss;
  grid_reduce4<kMThreads>(a.partials(), partials, counter,
                          [&](const ReducePartials& t) { *loss_out = t.ssn; });
}

template <class T>
__global__ void mesh_finalize_kernel(long long n, unsigned long long* __restrict__ acc,
                                     T* __restrict__ prop, T* __restrict__ diff) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    prop[k] = T(double((long long)acc[k]) / kFixM);
    diff[k] = T(double((long long)acc[n + k]) / kFixM);
    acc[k] = 0ull;
    acc[n + k] = 0ull;
  }
}

__global__ void mesh_intersect_kernel(MeshDev m, int n, const double* __restrict__ rays,
                                      double* __restrict__ t_out, int* __restrict__ tri_out) {
  MESH_SMEM;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double o[3] = {rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]};
    const double d[3] = {rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5]};
    double t = INFINITY, u, v;
    const int s = trace<false>(m, sn, stk, o, d, INFINITY, t, u, v);
    t_out[i] = s < 0 ? INFINITY : t;
    tri_out[i] = s < 0 ? -1 : m.orig[s];
  }
}

// ------------------------------------------------------------ wavefront
// The same estimator as mesh_pair_kernel, restructured into stages over
// SoA path state (north_star: "wavefront layout with coalesced SoA path
// state"): paths P = (nprop + 1) x pixels (proportional paths 0..nprop-1,
// path 0 also at theta_{t-1}; FD path nprop), then per depth
//   isect  : closest hit of every live path (all lanes traverse at once)
//   shade  : texel lookup, NEE sample + shadow-ray set-up, the BSDF values
//            for both parameter sets, Malley bounce; survivors re-queued
//   shadow : any-hit of the queued NEE rays; visible -> L += C
// and finally one thread per pixel forms the residual weights and scatters
// the stored adjoint data of the proportional paths.  Every per-path
// quantity is the megakernel's / oracle's (same operations, same order),
// so the results are bit-identical to both.
//
// Per-vertex adjoint fields (T, [v][field][PS]):
//   NCH 4 (metal 0): A[6] dSn[2] invfb[6] dSb[2] C[6]                 = 22
//   NCH 5          : A[6] invfb[6] C[6] dfn[2][3][3] dfb[2][3][3]      = 54
template <int NCH>
struct VF;
template <>
struct VF<4> {
  static constexpr int n = 22, A = 0, dSn = 6, invfb = 8, dSb = 14, C = 16;
};
template <>
struct VF<5> {
  static constexpr int n = 54, A = 0, invfb = 6, C = 12, dfn = 18, dfb = 36;
};

template <class T>
struct WF {
  double *ox, *oy, *oz, *dx, *dy, *dz;       // [P] ray
  double *ht, *hu, *hv;                       // [P] hit
  double *sox, *soy, *soz, *sdx, *sdy, *sdz, *stm;  // [P] shadow ray
  T *beta, *L, *E, *pendC;                    // [6][P]
  int *nv, *hslot, *q0, *q1, *sq;             // [P]
  int* vbase;                                 // [kMaxV][PS]
  T* vdat;                                    // [kMaxV][nvf][PS]
  unsigned int* cnt;                          // [2][kMaxV + 1]: queue / shadow counts
  int P, PS, npix, pix0, nprop, nvf;
};

template <class T>
size_t wf_bytes(int npix, int nprop, int nvf) {
  const size_t P = size_t(npix) * (nprop + 1), PS = size_t(npix) * nprop;
  return sizeof(double) * 16 * P + sizeof(T) * 24 * P + sizeof(int) * 5 * P +
         sizeof(int) * kMaxV * PS + sizeof(T) * kMaxV * nvf * PS +
         sizeof(unsigned int) * 2 * (kMaxV + 1) + 256 * 40;
}

template <class T>
WF<T> wf_carve(void* mem, int npix, int nprop, int nvf) {
  WF<T> w;
  char* c = static_cast<char*>(mem);
  auto take = [&](size_t bytes) {
    void* r = c;
    c += (bytes + 255) & ~size_t(255);
    return r;
  };
  w.npix = npix;
  w.nprop = nprop;
  w.nvf = nvf;
  w.P = npix * (nprop + 1);
  w.PS = npix * nprop;
  const size_t Pz = size_t(w.P);
  double** dd[] = {&w.ox, &w.oy, &w.oz, &w.dx, &w.dy, &w.dz, &w.ht, &w.hu, &w.hv,
                   &w.sox, &w.soy, &w.soz, &w.sdx, &w.sdy, &w.sdz, &w.stm};
  for (double** d : dd) *d = (double*)take(sizeof(double) * Pz);
  T** tt[] = {&w.beta, &w.L, &w.E, &w.pendC};
  for (T** t : tt) *t = (T*)take(sizeof(T) * 6 * Pz);
  int** ii[] = {&w.nv, &w.hslot, &w.q0, &w.q1, &w.sq};
  for (int** i : ii) *i = (int*)take(sizeof(int) * Pz);
  w.vbase = (int*)take(sizeof(int) * kMaxV * size_t(w.PS));
  w.vdat = (T*)take(sizeof(T) * kMaxV * size_t(nvf) * size_t(w.PS));
  w.cnt = (unsigned int*)take(sizeof(unsigned int) * 2 * (kMaxV + 1));
  return w;
}

// warp-aggregated append: slot in the queue, or -1 when !pred
__device__ __forceinline__ int enqueue(bool pred, unsigned int* counter) {
  const unsigned act = __activemask();
  const unsigned m = __ballot_sync(act, pred);
  const int lane = int(threadIdx.x & 31), leader = __ffs(act) - 1;
  unsigned base = 0;
  if (lane == leader && m) base = atomicAdd(counter, unsigned(__popc(m)));
  base = __shfl_sync(act, base, leader);
  return pred ? int(base) + __popc(m & ((1u << lane) - 1u)) : -1;
}

template <class T>
__device__ __forceinline__ T& vf(const WF<T>& w, int v, int f, int p) {
  return w.vdat[(size_t(v) * w.nvf + f) * size_t(w.PS) + p];
}

template <class T>
__global__ void __launch_bounds__(kMThreads) wf_gen_kernel(MeshK q, WF<T> w) {
  const double* V = q.view;
  for (int p = blockIdx.x * kMThreads + threadIdx.x; p < w.P; p += gridDim.x * kMThreads) {
    const int k = p / w.npix, pix = w.pix0 + (p - k * w.npix);
    const int px = pix % q.W, py = pix / q.W;
    double u[4];
    prng(q.key, uint32_t(pix), q.iteration, uint32_t(k), 0u, u);
    const double sx = ((double(px) + u[0]) / double(q.W)) * 2.0 - 1.0;
    const double sy = 1.0 - ((double(py) + u[1]) / double(q.H)) * 2.0;
    const double ax = sx * (V[12] * (double(q.W) / double(q.H))), ay = sy * V[12];
    double d[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) d[i] = (V[3 + i] + ax * V[6 + i]) + ay * V[9 + i];
    const double dl = sqrt(dot3d(d, d));
    w.ox[p] = V[0];
    w.oy[p] = V[1];
    w.oz[p] = V[2];
    w.dx[p] = d[0] / dl;
    w.dy[p] = d[1] / dl;
    w.dz[p] = d[2] / dl;
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      w.beta[size_t(j) * w.P + p] = T(1);
      w.L[size_t(j) * w.P + p] = T(0);
      w.E[size_t(j) * w.P + p] = T(0);
    }
    w.nv[p] = 0;
    w.q0[p] = p;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) w.cnt[0] = unsigned(w.P);
}

template <class T>
__global__ void __launch_bounds__(kMThreads, 8) wf_isect_kernel(MeshDev m, WF<T> w, int v) {
  MESH_SMEM;
  const int n = int(w.cnt[v]);
  const int* qin = (v & 1) ? w.q1 : w.q0;
  for (int i = blockIdx.x * kMThreads + threadIdx.x; i < n; i += gridDim.x * kMThreads) {
    const int p = qin[i];
    const double o[3] = {w.ox[p], w.oy[p], w.oz[p]}, d[3] = {w.dx[p], w.dy[p], w.dz[p]};
    double t = INFINITY, bu = 0.0, bv = 0.0;
    const int slot = trace_impl<false>(m, sn, o, d, INFINITY, t, bu, bv);
    w.hslot[p] = slot;
    w.ht[p] = t;
    w.hu[p] = bu;
    w.hv[p] = bv;
  }
}

template <class T, int NCH>
__global__ void __launch_bounds__(kMThreads)
    wf_shade_kernel(MeshK q, MeshDev m, WF<T> w, int v, const T* __restrict__ th0,
                    const T* __restrict__ th1) {
  using F = VF<NCH>;
  const double* V = q.view;
  const int maxv = int(V[24]);
  const int R2 = q.R * q.R;
  const int n = int(w.cnt[v]);
  const int* qin = (v & 1) ? w.q1 : w.q0;
  int* qout = (v & 1) ? w.q0 : w.q1;
  const double la = (V[15] - V[14]) * (V[17] - V[16]);
  const T* th[2] = {th0, th1};
  for (int i = blockIdx.x * kMThreads + threadIdx.x; i - int(threadIdx.x) < n;
       i += gridDim.x * kMThreads) {
    bool want_shadow = false, want_bounce = false;
    int p = -1;
    if (i < n) {
      p = qin[i];
      const int k = p / w.npix, pix = w.pix0 + (p - k * w.npix);
      const int slot = w.hslot[p];
      const bool store = p < w.PS;
      // parameter sets evaluated: path 0 (A) and the FD path at theta_t and
      // theta_{t-1}; the other proportional paths at theta_t only
      const int ns = (k == 0 || k == w.nprop) ? 2 : 1;
      // every stored field of vertex v is written exactly once below
      auto zero_nee = [&](int s) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          vf(w, v, F::A + s * 3 + c, p) = T(0);
          vf(w, v, F::C + s * 3 + c, p) = T(0);
        }
        if constexpr (NCH == 5) {
#pragma unroll
          for (int j = 0; j < 9; ++j) vf(w, v, VF<5>::dfn + s * 9 + j, p) = T(0);
        } else {
          vf(w, v, VF<4>::dSn + s, p) = T(0);
        }
      };
      auto zero_bounce = [&](int s) {
#pragma unroll
        for (int c = 0; c < 3; ++c) vf(w, v, F::invfb + s * 3 + c, p) = T(0);
        if constexpr (NCH == 5) {
#pragma unroll
          for (int j = 0; j < 9; ++j) vf(w, v, VF<5>::dfb + s * 9 + j, p) = T(0);
        } else {
          vf(w, v, VF<4>::dSb + s, p) = T(0);
        }
      };
      T beta[2][3];
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int c = 0; c < 3; ++c) beta[s][c] = w.beta[size_t(s * 3 + c) * w.P + p];
      if (slot < 0) {  // escaped: environment
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            if (s >= ns) break;
            const T e = beta[s][c] * T(V[21 + c]);
            w.E[size_t(s * 3 + c) * w.P + p] = e;
            w.L[size_t(s * 3 + c) * w.P + p] += e;
          }
      } else {
        const double o[3] = {w.ox[p], w.oy[p], w.oz[p]}, d[3] = {w.dx[p], w.dy[p], w.dz[p]};
        const double t = w.ht[p], bu = w.hu[p], bv = w.hv[p];
        const double* r = m.tri + size_t(kRec) * slot;
        const double x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
        double nn[3] = {r[9], r[10], r[11]};
        if (dot3d(nn, d) > 0.0) {
          nn[0] = -nn[0];
          nn[1] = -nn[1];
          nn[2] = -nn[2];
        }
        const double U = (r[12] + bu * r[14]) + bv * r[16];
        const double W_ = (r[13] + bu * r[15]) + bv * r[17];
        int tx = int(U * q.R), ty = int(W_ * q.R);
        tx = tx < 0 ? 0 : (tx > q.R - 1 ? q.R - 1 : tx);
        ty = ty < 0 ? 0 : (ty > q.R - 1 ? q.R - 1 : ty);
        const int pbase = __ldg(&m.obj[slot]) * NCH * R2 + ty * q.R + tx;
        w.nv[p] = v + 1;
        if (store) w.vbase[size_t(v) * w.PS + p] = pbase;
        bool nee_done = false, bounce_done = false;
        T base[2][3], rough[2], metal[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
#pragma unroll
          for (int c = 0; c < 3; ++c) base[s][c] = th[s][pbase + c * R2];
          rough[s] = th[s][pbase + 3 * R2];
          metal[s] = NCH == 5 ? th[s][pbase + 4 * R2] : T(0);
        }
        const double wo[3] = {-d[0], -d[1], -d[2]};
        const double xo[3] = {x[0] + kOff * nn[0], x[1] + kOff * nn[1], x[2] + kOff * nn[2]};
        double u[4];
        prng(q.key, uint32_t(pix), q.iteration, uint32_t(k), uint32_t(v * 256 + 1), u);
        const double lp[3] = {V[14] + u[0] * (V[15] - V[14]), V[13],
                              V[16] + u[1] * (V[17] - V[16])};
        double wl3[3] = {lp[0] - x[0], lp[1] - x[1], lp[2] - x[2]};
        const double d2 = dot3d(wl3, wl3);
        const double wl = sqrt(d2);
        wl3[0] /= wl;
        wl3[1] /= wl;
        wl3[2] /= wl;
        const double cx = dot3d(nn, wl3), cl = wl3[1];
        const T nT[3] = {T(nn[0]), T(nn[1]), T(nn[2])}, woT[3] = {T(wo[0]), T(wo[1]), T(wo[2])};
        if (cx > 0.0 && cl > 0.0 && dot3d(nn, wo) > 0.0) {
          want_shadow = true;
          const double gl = ((cx * cl) / d2) * la;
          const T wT[3] = {T(wl3[0]), T(wl3[1]), T(wl3[2])};
          nee_done = true;
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            if (s >= ns) break;
            T f[3];
            if constexpr (NCH == 5) {
              T df[3][3];
              bsdf_full<T>(base[s], metal[s], rough[s], nT, wT, woT, f, df);
              if (store)
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                  for (int kk = 0; kk < 3; ++kk) vf(w, v, F::dfn + s * 9 + c * 3 + kk, p) = df[c][kk];
            } else {
              T dS;
              bsdf_m0<T>(base[s], rough[s], nT, wT, woT, f, dS);
              if (store) vf(w, v, VF<4>::dSn + s, p) = dS;
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const T A = beta[s][c] * T(gl * V[18 + c]);
              const T Cc = A * f[c];
              if (store) {
                vf(w, v, F::A + s * 3 + c, p) = A;
                vf(w, v, F::C + s * 3 + c, p) = Cc;
              }
              w.pendC[size_t(s * 3 + c) * w.P + p] = Cc;
            }
          }
          w.sox[p] = xo[0];
          w.soy[p] = xo[1];
          w.soz[p] = xo[2];
          w.sdx[p] = wl3[0];
          w.sdy[p] = wl3[1];
          w.sdz[p] = wl3[2];
          w.stm[p] = wl - kOff;
        }
        if (!(v == maxv - 1 || dot3d(nn, wo) <= 0.0)) {
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
              prng(q.key, uint32_t(pix), q.iteration, uint32_t(k), uint32_t(v * 256 + 1) + j, c4);
            }
#pragma unroll
            for (int mm = 0; mm < 4; mm += 2) {
              if (got) break;
              const double a = 2.0 * c4[mm] - 1.0, b = 2.0 * c4[mm + 1] - 1.0;
              if (c4[mm] <= 1.0 && a * a + b * b < 1.0) {
                dx = a;
                dy = b;
                got = true;
              }
            }
          }
          const double dz = sqrt(fmax(0.0, 1.0 - (dx * dx + dy * dy)));
          if (dz > 0.0) {
            const double sign = copysign(1.0, nn[2]);
            const double aa = -1.0 / (sign + nn[2]);
            const double bb = nn[0] * nn[1] * aa;
            const double Tb[3] = {1.0 + sign * (nn[0] * nn[0]) * aa, sign * bb, -sign * nn[0]};
            const double Bb[3] = {bb, sign + (nn[1] * nn[1]) * aa, -nn[1]};
            const double wi[3] = {(dx * Tb[0] + dy * Bb[0]) + dz * nn[0],
                                  (dx * Tb[1] + dy * Bb[1]) + dz * nn[1],
                                  (dx * Tb[2] + dy * Bb[2]) + dz * nn[2]};
            const T wiT[3] = {T(wi[0]), T(wi[1]), T(wi[2])};
            bounce_done = true;
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              if (s >= ns) break;
              T f[3];
              if constexpr (NCH == 5) {
                T df[3][3];
                bsdf_full<T>(base[s], metal[s], rough[s], nT, wiT, woT, f, df);
                if (store)
#pragma unroll
                  for (int c = 0; c < 3; ++c)
#pragma unroll
                    for (int kk = 0; kk < 3; ++kk)
                      vf(w, v, F::dfb + s * 9 + c * 3 + kk, p) = df[c][kk];
              } else {
                T dS;
                bsdf_m0<T>(base[s], rough[s], nT, wiT, woT, f, dS);
                if (store) vf(w, v, VF<4>::dSb + s, p) = dS;
              }
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                if (store) vf(w, v, F::invfb + s * 3 + c, p) = f[c] != T(0) ? T(1) / f[c] : T(0);
                w.beta[size_t(s * 3 + c) * w.P + p] = beta[s][c] * (f[c] * T(kPiM));
              }
            }
            w.ox[p] = xo[0];
            w.oy[p] = xo[1];
            w.oz[p] = xo[2];
            w.dx[p] = wi[0];
            w.dy[p] = wi[1];
            w.dz[p] = wi[2];
            want_bounce = true;
          }
        }
        if (store)
          for (int s = 0; s < ns; ++s) {
            if (!nee_done) zero_nee(s);
            if (!bounce_done) zero_bounce(s);
          }
      }
    }
    const int qs = enqueue(want_shadow, &w.cnt[kMaxV + 1 + v]);
    if (qs >= 0) w.sq[qs] = p;
    const int qb = enqueue(want_bounce, &w.cnt[v + 1]);
    if (qb >= 0) qout[qb] = p;
  }
}

template <class T, int NCH>
__global__ void __launch_bounds__(kMThreads, 8) wf_shadow_kernel(MeshDev m, WF<T> w, int v) {
  using F = VF<NCH>;
  MESH_SMEM;
  const int n = int(w.cnt[kMaxV + 1 + v]);
  for (int i = blockIdx.x * kMThreads + threadIdx.x; i < n; i += gridDim.x * kMThreads) {
    const int p = w.sq[i];
    const double o[3] = {w.sox[p], w.soy[p], w.soz[p]}, d[3] = {w.sdx[p], w.sdy[p], w.sdz[p]};
    double ts, tu, tv;
    if (trace_impl<true>(m, sn, o, d, w.stm[p], ts, tu, tv) < 0) {
      const int k = p / w.npix;
      const int nj = (k == 0 || k == w.nprop) ? 6 : 3;
      for (int j = 0; j < nj; ++j) w.L[size_t(j) * w.P + p] += w.pendC[size_t(j) * w.P + p];
    } else if (p < w.PS) {  // occluded: no NEE data at this vertex
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        vf(w, v, F::A + j, p) = T(0);
        vf(w, v, F::C + j, p) = T(0);
      }
      if constexpr (NCH == 5) {
        for (int j = 0; j < 18; ++j) vf(w, v, VF<5>::dfn + j, p) = T(0);
      } else {
        vf(w, v, VF<4>::dSn, p) = T(0);
        vf(w, v, VF<4>::dSn + 1, p) = T(0);
      }
    }
  }
}

// adjoint of stored path p (megakernel `scatter` / oracle ms_scatter)
template <class T, int NCH>
__device__ __noinline__ void wf_scatter(const WF<T>& w, int p, int s, const T wt[3], int R2,
                                        unsigned long long* __restrict__ acc) {
  using F = VF<NCH>;
  T Q[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) Q[c] = w.E[size_t(s * 3 + c) * w.P + p];
  for (int v = w.nv[p] - 1; v >= 0; --v) {
    const int base = w.vbase[size_t(v) * w.PS + p];
    if constexpr (NCH == 5) {
      T gm = T(0), gr = T(0);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const T A = vf(w, v, F::A + s * 3 + c, p), fb = vf(w, v, F::invfb + s * 3 + c, p);
        const int dn = F::dfn + s * 9 + c * 3, db = F::dfb + s * 9 + c * 3;
        const T gb = wt[c] * (A * vf(w, v, dn, p) + Q[c] * (fb * vf(w, v, db, p)));
        atomicAdd(&acc[base + c * R2], fixq(double(gb)));
        gm += wt[c] * (A * vf(w, v, dn + 1, p) + Q[c] * (fb * vf(w, v, db + 1, p)));
        gr += wt[c] * (A * vf(w, v, dn + 2, p) + Q[c] * (fb * vf(w, v, db + 2, p)));
      }
      atomicAdd(&acc[base + 3 * R2], fixq(double(gr)));
      atomicAdd(&acc[base + 4 * R2], fixq(double(gm)));
    } else {
      const T dSn = vf(w, v, F::dSn + s, p), dSb = vf(w, v, F::dSb + s, p);
      T gr = T(0);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const T A = vf(w, v, F::A + s * 3 + c, p), ifb = vf(w, v, F::invfb + s * 3 + c, p);
        const T gb = wt[c] * ((A / T(kPiM)) + Q[c] * (ifb / T(kPiM)));
        atomicAdd(&acc[base + c * R2], fixq(double(gb)));
        gr += wt[c] * (A * dSn + Q[c] * (ifb * dSb));
      }
      atomicAdd(&acc[base + 3 * R2], fixq(double(gr)));
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) Q[c] = Q[c] + vf(w, v, F::C + s * 3 + c, p);
  }
}

constexpr int kMaxProp = 8;

template <class T, int NCH>
__global__ void __launch_bounds__(kMThreads)
    wf_scatter_kernel(MeshK q, WF<T> w, const T* __restrict__ target_img,
                      unsigned long long* __restrict__ acc, long long np,
                      ReducePartials* partials, unsigned int* counter, double* loss_out) {
  const int npix_img = q.W * q.H;
  const int R2 = q.R * q.R;
  const int n = w.nprop;
  const T scale = T(2.0 / (n * (n - 1.0)));
  double loss = 0.0;
  for (int i = blockIdx.x * kMThreads + threadIdx.x; i < w.npix; i += gridDim.x * kMThreads) {
    const int pix = w.pix0 + i;
    const int pc = n * w.npix + i;
    T r[kMaxProp][3], wC0[3], wC1[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const T Is = target_img[size_t(c) * npix_img + pix];
      for (int j = 0; j < n; ++j) r[j][c] = w.L[size_t(c) * w.P + j * w.npix + i] - Is;
      wC0[c] = T(2) * (w.L[size_t(c) * w.P + pc] - Is);
      wC1[c] = T(-2) * (w.L[size_t(3 + c) * w.P + pc] - Is);
      T lp = T(0);
      for (int a = 0; a < n; ++a)
        for (int b = a + 1; b < n; ++b) lp += r[a][c] * r[b][c];
      loss += double(lp * scale);
    }
    for (int j = 0; j < n; ++j) {
      T wt[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        T a = T(0);
        bool first = true;
        for (int k = 0; k < n; ++k) {
          if (k == j) continue;
          a = first ? r[k][c] : a + r[k][c];
          first = false;
        }
        wt[c] = a * scale;
      }
      wf_scatter<T, NCH>(w, j * w.npix + i, 0, wt, R2, acc);
    }
    wf_scatter<T, NCH>(w, i, 0, wC0, R2, acc + np);
    wf_scatter<T, NCH>(w, i, 1, wC1, R2, acc + np);
  }
  Acc a;
  a.ssn = loss;
  grid_reduce4<kMThreads>(a.partials(), partials, counter,
                          [&](const ReducePartials& t) { *loss_out = t.ssn; });
}

MeshDev dev_of(const mg_mesh_scene* s) {
  MeshDev m;
  m.tri = s->tri;
  m.orig = s->orig;
  m.obj = s->obj;
  m.nodes = s->nodes;
  m.nnodes = s->nnodes;
  return m;
}

MeshK make_k(const mg_mesh_scene* s, int W, int H, const double* view, uint64_t key,
             uint32_t it) {
  MeshK q;
  q.W = W;
  q.H = H;
  q.R = s->R;
  q.nobj = s->nobj;
  q.nch = s->nch;
  q.row0 = 0;
  q.row1 = H;
  for (int i = 0; i < 25; ++i) q.view[i] = view[i];
  q.key = key;
  q.iteration = it;
  return q;
}

}  // namespace
template <class T, int NCH>
int wavefront_pair(mg_ctx* ctx, mg_mesh_scene* s, const MeshK& q, int nprop, const T* target_img,
                   const T* now, const T* prev, unsigned long long* acc, long long np,
                   double* loss_out) {
  const int npix = q.W * (q.row1 - q.row0);
  if (npix == 0) {
    MG_CUDA_TRY(cudaMemsetAsync(loss_out, 0, sizeof(double), ctx->stream));
    return MG_OK;
  }
  if (int64_t(npix) * (nprop + 1) > 0x7fffffffLL) return fail(MG_EINVAL, "mesh scene: image too large");
  const size_t need = wf_bytes<T>(npix, nprop, VF<NCH>::n);
  if (need > s->wf_cap) {
    MG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    cudaFree(s->wf);
    s->wf = nullptr;
    s->wf_cap = 0;
    MG_CUDA_TRY(cudaMalloc(&s->wf, need));
    s->wf_cap = need;
  }
  WF<T> w = wf_carve<T>(s->wf, npix, nprop, VF<NCH>::n);
  w.pix0 = q.row0 * q.W;
  const MeshDev m = dev_of(s);
  MG_CUDA_TRY(cudaMemsetAsync(w.cnt, 0, sizeof(unsigned int) * 2 * (kMaxV + 1), ctx->stream));
  const int grid = grid_for(ctx, w.P, kMThreads, 8);
  wf_gen_kernel<T><<<grid, kMThreads, 0, ctx->stream>>>(q, w);
  MG_LAUNCH_CHECK(ctx);
  const int maxv = int(q.view[24]);
  for (int v = 0; v < maxv; ++v) {
    wf_isect_kernel<T><<<grid, kMThreads, 0, ctx->stream>>>(m, w, v);
    MG_LAUNCH_CHECK(ctx);
    wf_shade_kernel<T, NCH><<<grid, kMThreads, 0, ctx->stream>>>(q, m, w, v, now, prev);
    MG_LAUNCH_CHECK(ctx);
    wf_shadow_kernel<T, NCH><<<grid, kMThreads, 0, ctx->stream>>>(m, w, v);
    MG_LAUNCH_CHECK(ctx);
  }
  wf_scatter_kernel<T, NCH><<<grid_for(ctx, npix, kMThreads, 8), kMThreads, 0, ctx->stream>>>(
      q, w, target_img, acc, np, ctx->partials, ctx->counter, loss_out);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

}  // namespace mg

using namespace mg;

extern "C" {

int mg_meshscene_create(mg_ctx* ctx, int32_t tri_count, const double* tri, const int32_t* obj,
                        int32_t nobj, int32_t tex_res, int32_t channels, mg_mesh_scene** out) {
  if (!ctx || !tri || !obj || !out) return fail(MG_EINVAL, "mg_meshscene_create: null argument");
  if (channels != 4 && channels != 5)
    return fail(MG_EINVAL, "mg_meshscene_create: channels must be 4 (base rgb, roughness) or 5 "
                           "(+ metalness)");
  if (tri_count < 1 || nobj < 1 || tex_res < 1)
    return fail(MG_EINVAL, "mg_meshscene_create: bad sizes");
  if (tri_count > (1 << 27)) return fail(MG_EINVAL, "mg_meshscene_create: more than 2^27 triangles");
  if (int64_t(nobj) * channels * tex_res * tex_res > 0x7fffffffLL)
    return fail(MG_EINVAL, "mg_meshscene_create: parameter count exceeds 2^31");
  for (int k = 0; k < tri_count; ++k)
    if (obj[k] < 0 || obj[k] >= nobj) return fail(MG_EINVAL, "mg_meshscene_create: bad object id");
  Builder B;
  B.tri = tri;
  const size_t T = size_t(tri_count);
  B.blo.resize(3 * T);
  B.bhi.resize(3 * T);
  B.cen.resize(3 * T);
  B.idx.resize(T);
  double slo[3] = {INFINITY, INFINITY, INFINITY}, shi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (size_t k = 0; k < T; ++k) {
    const double* r = tri + kRec * k;
    for (int a = 0; a < 3; ++a) {
      const double p0 = r[a], p1 = r[a] + r[3 + a], p2 = r[a] + r[6 + a];
      const double lo = std::min(p0, std::min(p1, p2)), hi = std::max(p0, std::max(p1, p2));
      B.blo[3 * k + a] = lo;
      B.bhi[3 * k + a] = hi;
      B.cen[3 * k + a] = 0.5 * (lo + hi);
      slo[a] = std::min(slo[a], lo);
      shi[a] = std::max(shi[a], hi);
    }
    B.idx[k] = int(k);
  }
  B.nodes.reserve(2 * T);
  B.build(0, tri_count, 0);
  if (B.too_deep) return fail(MG_EINVAL, "mg_meshscene_create: BVH deeper than the traversal stack");
  // Internal nodes in breadth-first order (the top levels become nodes
  // [0, kSmemNodes) for the shared-memory stage); each stores its two
  // children's boxes.  A single-leaf tree gets a root whose second child is
  // an empty box.
  const double diag = sqrt((shi[0] - slo[0]) * (shi[0] - slo[0]) +
                           (shi[1] - slo[1]) * (shi[1] - slo[1]) +
                           (shi[2] - slo[2]) * (shi[2] - slo[2]));
  const float pad = float(1e-5 * diag + 1e-7);
  std::vector<int> order, label(B.nodes.size(), -1);
  if (B.nodes[0].left >= 0) {
    order.push_back(0);
    label[0] = 0;
    for (size_t h = 0; h < order.size(); ++h) {
      const TmpNode& nd = B.nodes[size_t(order[h])];
      for (int c : {nd.left, nd.right})
        if (B.nodes[size_t(c)].left >= 0) {
          label[size_t(c)] = int(order.size());
          order.push_back(c);
        }
    }
  }
  auto child_ref = [&](int c) {
    const TmpNode& nd = B.nodes[size_t(c)];
    return nd.left >= 0 ? label[size_t(c)] : ~(nd.first * 8 + nd.count);
  };
  auto box = [&](int c, float* lo, float* hi) {
    const TmpNode& nd = B.nodes[size_t(c)];
    for (int a = 0; a < 3; ++a) {
      lo[a] = nextafterf(float(nd.lo[a]), -INFINITY) - pad;
      hi[a] = nextafterf(float(nd.hi[a]), INFINITY) + pad;
    }
  };
  auto ibits = [](int v) {
    float f;
    memcpy(&f, &v, 4);
    return f;
  };
  const int nn = order.empty() ? 1 : int(order.size());
  std::vector<float4> nodes(4 * size_t(nn));
  for (int i = 0; i < nn; ++i) {
    float l0[3], h0[3], l1[3] = {1.0f, 1.0f, 1.0f}, h1[3] = {-1.0f, -1.0f, -1.0f};
    int r0, r1 = ~0;  // empty leaf
    if (order.empty()) {
      box(0, l0, h0);
      r0 = child_ref(0);
    } else {
      const TmpNode& nd = B.nodes[size_t(order[size_t(i)])];
      box(nd.left, l0, h0);
      box(nd.right, l1, h1);
      r0 = child_ref(nd.left);
      r1 = child_ref(nd.right);
    }
    nodes[4 * size_t(i)] = make_float4(l0[0], l0[1], l0[2], h0[0]);
    nodes[4 * size_t(i) + 1] = make_float4(h0[1], h0[2], l1[0], l1[1]);
    nodes[4 * size_t(i) + 2] = make_float4(l1[2], h1[0], h1[1], h1[2]);
    nodes[4 * size_t(i) + 3] = make_float4(ibits(r0), ibits(r1), 0.0f, 0.0f);
  }
  std::vector<double> stri(kRec * T);
  std::vector<int> sorig(T), sobj(T);
  for (size_t s = 0; s < T; ++s) {
    const int k = B.idx[s];
    memcpy(&stri[kRec * s], tri + kRec * size_t(k), sizeof(double) * kRec);
    sorig[s] = k;
    sobj[s] = obj[k];
  }
  mg_mesh_scene* sc = new mg_mesh_scene();
  sc->T = tri_count;
  sc->nobj = nobj;
  sc->nch = channels;
  sc->R = tex_res;
  sc->nnodes = nn;
  sc->depth = B.max_depth;
  cudaError_t e = cudaMalloc(&sc->tri, sizeof(double) * stri.size());
  if (e == cudaSuccess) e = cudaMalloc(&sc->orig, sizeof(int) * T);
  if (e == cudaSuccess) e = cudaMalloc(&sc->obj, sizeof(int) * T);
  if (e == cudaSuccess) e = cudaMalloc(&sc->nodes, sizeof(float4) * nodes.size());
  if (e == cudaSuccess) e = cudaMalloc(&sc->work, sizeof(unsigned int));
  if (e == cudaSuccess)
    e = cudaMemcpy(sc->tri, stri.data(), sizeof(double) * stri.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(sc->orig, sorig.data(), sizeof(int) * T, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(sc->obj, sobj.data(), sizeof(int) * T, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(sc->nodes, nodes.data(), sizeof(float4) * nodes.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(sc->tri);
    cudaFree(sc->orig);
    cudaFree(sc->obj);
    cudaFree(sc->nodes);
    cudaFree(sc->work);
    delete sc;
    return cuda_fail(e, "mg_meshscene_create");
  }
  *out = sc;
  return MG_OK;
}

int mg_meshscene_destroy(mg_mesh_scene* s) {
  if (!s) return MG_OK;
  cudaFree(s->tri);
  cudaFree(s->orig);
  cudaFree(s->obj);
  cudaFree(s->nodes);
  cudaFree(s->work);
  cudaFree(s->wf);
  delete s;
  return MG_OK;
}

int mg_meshscene_info(const mg_mesh_scene* s, int32_t* nodes, int32_t* depth, int64_t* params) {
  if (!s) return fail(MG_EINVAL, "mg_meshscene_info: null scene");
  if (nodes) *nodes = s->nnodes;
  if (depth) *depth = s->depth;
  if (params) *params = int64_t(s->nobj) * s->nch * s->R * s->R;
  return MG_OK;
}

int mg_meshscene_intersect(mg_ctx* ctx, const mg_mesh_scene* s, int32_t n, const double* rays,
                           double* t_out, int32_t* tri_out) {
  if (!ctx || !s || (n > 0 && (!rays || !t_out || !tri_out)))
    return fail(MG_EINVAL, "mg_meshscene_intersect: null argument");
  if (n <= 0) return MG_OK;
  const int grid = grid_for(ctx, n, kMThreads, 8);
  mesh_intersect_kernel<<<grid, kMThreads, 0, ctx->stream>>>(dev_of(s), n, rays, t_out, tri_out);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

static int check_view(const double* view) {
  if (!view) return fail(MG_EINVAL, "mesh scene: null view");
  const int maxv = int(view[24]);
  if (maxv < 1 || maxv > kMaxV) return fail(MG_EINVAL, "mesh scene: max_vertices must lie in [1, 8]");
  return MG_OK;
}

int mg_meshscene_render(mg_ctx* ctx, const mg_mesh_scene* s, int32_t dtype, int32_t W, int32_t H,
                        const double* view, int32_t spp, uint64_t key, const void* theta,
                        void* img) {
  if (!ctx || !s || !theta || !img) return fail(MG_EINVAL, "mg_meshscene_render: null argument");
  if (W < 1 || H < 1 || spp < 1) return fail(MG_EINVAL, "mg_meshscene_render: bad sizes");
  int st = check_view(view);
  if (st) return st;
  const MeshK q = make_k(s, W, H, view, key, 0xffffffffu);
  const int grid = grid_for(ctx, int64_t(W) * H, kMThreads, 4);
  const bool five = s->nch == 5;
  if (dtype == MG_F64 && five)
    mesh_render_kernel<double, 5><<<grid, kMThreads, 0, ctx->stream>>>(
        q, dev_of(s), spp, (const double*)theta, (double*)img);
  else if (dtype == MG_F64)
    mesh_render_kernel<double, 4><<<grid, kMThreads, 0, ctx->stream>>>(
        q, dev_of(s), spp, (const double*)theta, (double*)img);
  else if (dtype == MG_F32 && five)
    mesh_render_kernel<float, 5><<<grid, kMThreads, 0, ctx->stream>>>(
        q, dev_of(s), spp, (const float*)theta, (float*)img);
  else if (dtype == MG_F32)
    mesh_render_kernel<float, 4><<<grid, kMThreads, 0, ctx->stream>>>(
        q, dev_of(s), spp, (const float*)theta, (float*)img);
  else
    return fail(MG_EINVAL, "mg_meshscene_render: unknown dtype");
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

int mg_meshscene_sample_pair(mg_ctx* ctx, mg_mesh_scene* s, int32_t dtype, int32_t W,
                             int32_t H, const double* view, const void* target_img,
                             const void* now, const void* prev, uint64_t key, uint32_t iteration,
                             int32_t row0, int32_t row1, int32_t prop_paths, void* accum,
                             void* prop, void* diff, double* loss_out) {
  if (!ctx || !s || !target_img || !now || !prev || !accum || !prop || !diff || !loss_out)
    return fail(MG_EINVAL, "mg_meshscene_sample_pair: null argument");
  if (prop_paths < 2 || prop_paths > kMaxProp)
    return fail(MG_EINVAL, "mg_meshscene_sample_pair: prop_paths must lie in [2, 8]");
  if (W < 1 || H < 1) return fail(MG_EINVAL, "mg_meshscene_sample_pair: bad sizes");
  if (row0 < 0 || row1 > H || row0 > row1)
    return fail(MG_EINVAL, "mg_meshscene_sample_pair: bad rows");
  int st = check_view(view);
  if (st) return st;
  MeshK q = make_k(s, W, H, view, key, iteration);
  q.row0 = row0;
  q.row1 = row1;
  const long long np = (long long)s->nobj * s->nch * s->R * s->R;
  const int grid = grid_for(ctx, int64_t(W) * (row1 - row0) + 1, kMThreads, 4);
  unsigned long long* acc = (unsigned long long*)accum;
  // the megakernel implements the configs[3] form (4 channels, 2 proportional paths)
  if (g_mesh_megakernel && s->nch == 4 && prop_paths == 2) {
    MG_CUDA_TRY(cudaMemsetAsync(s->work, 0, sizeof(unsigned int), ctx->stream));
    if (dtype == MG_F64)
      mesh_pair_kernel<double><<<grid, kMThreads, 0, ctx->stream>>>(
          q, dev_of(s), (const double*)target_img, (const double*)now, (const double*)prev, acc,
          np, s->work, ctx->partials, ctx->counter, loss_out);
    else if (dtype == MG_F32)
      mesh_pair_kernel<float><<<grid, kMThreads, 0, ctx->stream>>>(
          q, dev_of(s), (const float*)target_img, (const float*)now, (const float*)prev, acc, np,
          s->work, ctx->partials, ctx->counter, loss_out);
    else
      return fail(MG_EINVAL, "mg_meshscene_sample_pair: unknown dtype");
    MG_LAUNCH_CHECK(ctx);
  } else if (dtype == MG_F64 && s->nch == 5) {
    st = wavefront_pair<double, 5>(ctx, s, q, prop_paths, (const double*)target_img,
                                   (const double*)now, (const double*)prev, acc, np, loss_out);
  } else if (dtype == MG_F64) {
    st = wavefront_pair<double, 4>(ctx, s, q, prop_paths, (const double*)target_img,
                                   (const double*)now, (const double*)prev, acc, np, loss_out);
  } else if (dtype == MG_F32 && s->nch == 5) {
    st = wavefront_pair<float, 5>(ctx, s, q, prop_paths, (const float*)target_img,
                                  (const float*)now, (const float*)prev, acc, np, loss_out);
  } else if (dtype == MG_F32) {
    st = wavefront_pair<float, 4>(ctx, s, q, prop_paths, (const float*)target_img,
                                  (const float*)now, (const float*)prev, acc, np, loss_out);
  } else {
    return fail(MG_EINVAL, "mg_meshscene_sample_pair: unknown dtype");
  }
  if (st) return st;
  const int fgrid = grid_for(ctx, np, 256, 8);
  if (dtype == MG_F64)
    mesh_finalize_kernel<double><<<fgrid, 256, 0, ctx->stream>>>(np, acc, (double*)prop,
                                                                 (double*)diff);
  else
    mesh_finalize_kernel<float><<<fgrid, 256, 0, ctx->stream>>>(np, acc, (float*)prop,
                                                                (float*)diff);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

}  // extern "C"
