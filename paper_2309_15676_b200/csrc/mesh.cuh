// Shared declarations of the triangle-mesh renderer (F1 slices 3-4,
// BASELINE.json configs[3] and [4]): the scene object, the
// kernel parameter blocks and the device building blocks — BVH node layout
// and traversal, fp64 Moller-Trumbore, Philox addressing, the principled
// BSDF and its parameter derivatives.  Oracle: oracle/metagrad_oracle.c
// mgo_mesh*_* (the reference has no renderer).
//
//   mesh_bvh.cu        host BVH build, scene create / destroy / info
//   mesh_megakernel.cu one-thread-per-pixel path (configs[3] form), render,
//                      ray-query entry point
//   mesh_wavefront.cu  the default wavefront sample pair (configs[3] and [4])
#pragma once

#include <math.h>
#include <stdint.h>

#include <climits>

#include "mg_common.cuh"
#include "philox.cuh"

struct mg_mesh_scene {
  int T = 0, nobj = 0, R = 0, nnodes = 0, depth = 0, nch = 4;
  double* tri = nullptr;   // [T][18] in BVH order
  float4* tri32 = nullptr; // [T][3] fp32 v0 e1 e2 (fp32-mode traversal), BVH order
  int* orig = nullptr;     // [T] original triangle index
  int* obj = nullptr;      // [T] object id (BVH order)
  float4* nodes = nullptr; // [kNodeF4 * nnodes]: BVH4 (see NodeW)
  float4* nodes8 = nullptr; // [kNode8F4 * nnodes8]: BVH8 of the fp32 persistent traversal
  float4* nodesq = nullptr; // [kNodeQF4 * nnodes]: the BVH4 with quantised child boxes
  int nnodes8 = 0, depth8 = 0;
  unsigned int* work = nullptr;  // pixel work counter of the pair kernel
  void* wf = nullptr;            // wavefront path state (grow-only)
  size_t wf_cap = 0;
  // texel-major parameter copies in the workspace (mg_meshscene_set_prev_reuse)
  bool prev_reuse = false;
  const void* last_now = nullptr;  // `now` of the previous wavefront call ...
  int last_now_slot = -1;          // ... the copy slot holding it (-1: none)
  int last_dtype = -1;
  unsigned int* last_cnt = nullptr;  // queue counters of the last wavefront call
  // caller-owned bit per texel cell, set by the accumulator-keeping sample
  // pair for every cell it adds to (mg_meshscene_set_touch_map)
  unsigned int* touch = nullptr;
};

namespace mg {
// mg_set_option("mesh_megakernel", 1): one-thread-per-pixel megakernel
// instead of the default wavefront stages (A/B comparison; identical results)
extern bool g_mesh_megakernel;
// mg_set_option("mesh_persistent", 0): fp32 isect / shadow stages with the
// grid-stride one-ray-per-thread traversal instead of the persistent warp loop
// bit 0: isect, bit 1: shadow; -1 (default): both.  (With the local-memory
// stack and fp32 nodes, the persistent isect lost on configs[3]'s 5.9k-node
// BVH, +0.035 ms; with the shared-memory stack and quantised nodes it wins
// there too, 1.211 -> 1.143 ms.)
extern int g_mesh_persistent;
// mg_set_option("mesh_tail", d): fp32 wavefront depths >= d (0-based) run in
// one wf_tail_kernel launch; 0 = never; -1 (default): the last kMeshTailDepths
// depths (from depth 1 at the earliest) — measured best on configs[3] (depth
// 6: tail from 2) and configs[4] (depth 8: 3 and 4 equal)
extern int g_mesh_tail;
constexpr int kMeshTailDepths = 4;
// mg_set_option("mesh_smem_stack", 1): the persistent BVH4 traversals keep
// their stack in shared memory ([entry][thread], conflict-free) instead of
// staging the top nodes there
extern bool g_mesh_smem_stack;
// mg_set_option("mesh_qnodes", 0): the shared-memory-stack traversal reads
// the full fp32 BVH4 nodes instead of the quantised 64-byte copies
extern bool g_mesh_qnodes;
// mg_set_option("mesh_bvh8", 0): the persistent fp32 traversals walk the
// BVH4 instead of the BVH8
extern bool g_mesh_bvh8;
// mg_set_option("mesh_scatter_aggregate", 1): warp-aggregated adjoint
// scatter (__match_any_sync per texel cell).  Off by default: the paths of
// one warp almost never share a texel at configs[3]/[4] texture densities,
// so the match costs more than it saves (configs[4] 9.05 -> 9.14 ms,
// configs[3] unchanged; tools/mesh_ab_options.py, bit-identical)
extern bool g_mesh_scatter_agg;
// mg_set_option("bvh_leaf_size", k): maximum triangles per BVH leaf (1..7),
// applied to scenes created afterwards
extern int g_bvh_leaf;
// mg_set_option("bvh_sah_axes", 1 | 3): binned-SAH split candidates on the
// longest centroid axis only, or on all three (default), for scenes created
// afterwards
extern int g_bvh_axes;
// mg_set_option("bvh_bins", n): SAH bins per axis (2..64, default 32:
// configs[4] 6.80 -> 6.77 ms against 16, 6.92 with 8; configs[3] +-0)
extern int g_bvh_bins;

namespace mesh {

constexpr int kMThreads = 128;
constexpr int kMaxV = 8;
constexpr int kRec = 18;
constexpr int kSmemNodes = 128;  // top BVH4 levels staged in shared memory (16 KB)
constexpr int kStackDepth = 64;  // traversal stack per thread (local memory)
constexpr double kTMin = 1e-9, kOff = 1e-6;
constexpr double kPiM = 3.14159265358979323846;
constexpr double kFixM = 1099511627776.0;  // 2^40

// ------------------------------------------------------------ device
struct MeshDev {
  const double* __restrict__ tri;
  const float4* __restrict__ tri32;  // [T][3]: v0, e1, e2 in fp32 (fast-mode traversal)
  const int* __restrict__ orig;
  const int* __restrict__ obj;
  const float4* __restrict__ nodes;
  int nnodes;
  const float4* __restrict__ nodes8;
  int nnodes8;
  const float4* __restrict__ nodesq;
};

struct MeshK {
  int W, H, R, nobj, nch;
  int row0, row1;
  double view[25];
  uint64_t key;
  uint32_t iteration;
  const uint32_t* it_offset;  // device iteration offset or null (mg_ctx_set_iteration_offset)
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

// BVH4 node = the boxes of up to four children in SoA form (128 B, eight
// float4): lo.x[4] lo.y[4] lo.z[4] hi.x[4] hi.y[4] hi.z[4] ref[4] pad;
// ref >= 0: internal node, ref < 0: leaf with triangles [first, first +
// count), ~ref = first * 8 + count; empty slots have an inverted box.
// One 128-byte fetch per traversal step tests all four children.
#ifndef MG_ANY_SORT
#define MG_ANY_SORT 0
#endif
constexpr int kNodeF4 = 8;
constexpr int kNodeQF4 = 4;  // quantised BVH4 node: 64 bytes
struct NodeW {
  float4 lx, ly, lz, hx, hy, hz, ref;
};

template <bool STAGED = true>
__device__ __forceinline__ NodeW load_node(const MeshDev& m, const float4* sn, int i) {
  const bool shared = STAGED && i < kSmemNodes;
  const float4* src = shared ? sn + kNodeF4 * i : m.nodes + size_t(kNodeF4) * i;
  NodeW n;
  if (shared) {
    n.lx = src[0];
    n.ly = src[1];
    n.lz = src[2];
    n.hx = src[3];
    n.hy = src[4];
    n.hz = src[5];
    n.ref = src[6];
  } else {
    n.lx = __ldg(src);
    n.ly = __ldg(src + 1);
    n.lz = __ldg(src + 2);
    n.hx = __ldg(src + 3);
    n.hy = __ldg(src + 4);
    n.hz = __ldg(src + 5);
    n.ref = __ldg(src + 6);
  }
  return n;
}

__device__ __forceinline__ float f4c(const float4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

// Slab test in FMA form: t = box * inv - o * inv (ooi = o * inv once per
// ray, one FFMA per plane).  The rounding of ooi is of the order of the
// fp32 rounding of the origin itself, which the outward box padding
// (1e-5 of the scene diagonal) already absorbs.
__device__ __forceinline__ bool slab6(float lx, float ly, float lz, float hx, float hy, float hz,
                                      const float ooi[3], const float inv[3], float tmax,
                                      float& tnear) {
  const float tx0 = fmaf(lx, inv[0], -ooi[0]), tx1 = fmaf(hx, inv[0], -ooi[0]);
  const float ty0 = fmaf(ly, inv[1], -ooi[1]), ty1 = fmaf(hy, inv[1], -ooi[1]);
  const float tz0 = fmaf(lz, inv[2], -ooi[2]), tz1 = fmaf(hz, inv[2], -ooi[2]);
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
// The traversal stack is a per-thread local array (a shared-memory stack
// measured slower: it cut occupancy).
template <bool ANY>
__device__ __forceinline__ int trace_impl(const MeshDev& m, const float4* sn, const double o[3],
                                          const double d[3], double tmax, double& t_out,
                                          double& u_out, double& v_out) {
  float ooi[3], inv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float dk = float(d[k]);
    inv[k] = 1.0f / (fabsf(dk) > 1e-20f ? dk : copysignf(1e-20f, dk));
    ooi[k] = float(o[k]) * inv[k];
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
      MG_DCHECK(node < m.nnodes && sp + 4 <= kStackDepth);
      const NodeW n = load_node(m, sn, node);
      // (entry distance, child) of the hit children, sorted ascending by a
      // 4-input sorting network (misses carry +inf)
      float tk[4];
      int ck[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float tc;
        const bool h = slab6(f4c(n.lx, c), f4c(n.ly, c), f4c(n.lz, c), f4c(n.hx, c), f4c(n.hy, c),
                             f4c(n.hz, c), ooi, inv, bestf, tc);
        tk[c] = h ? tc : INFINITY;
        ck[c] = __float_as_int(f4c(n.ref, c));
      }
      auto cx = [&](int a, int b) {
        if (tk[b] < tk[a]) {
          const float tt = tk[a];
          tk[a] = tk[b];
          tk[b] = tt;
          const int cc = ck[a];
          ck[a] = ck[b];
          ck[b] = cc;
        }
      };
      if (!ANY || MG_ANY_SORT) {  // any-hit rays need no front-to-back order
        cx(0, 1);
        cx(2, 3);
        cx(0, 2);
        cx(1, 3);
        cx(1, 2);
      }
      if (ANY && !MG_ANY_SORT) {
        int nx = 0;
        bool have = false;
#pragma unroll
        for (int c = 3; c >= 0; --c) {
          if (tk[c] == INFINITY) continue;
          if (have) stack[sp++] = nx;
          nx = ck[c];
          have = true;
        }
        if (have) {
          node = nx;
          continue;
        }
      } else if (tk[0] != INFINITY) {
        if (tk[3] != INFINITY) stack[sp++] = ck[3];
        if (tk[2] != INFINITY) stack[sp++] = ck[2];
        if (tk[1] != INFINITY) stack[sp++] = ck[1];
        node = ck[0];
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
__device__ __noinline__ int trace(const MeshDev& m, const float4* sn, const double o[3],
                                  const double d[3], double tmax, double& t_out, double& u_out,
                                  double& v_out) {
  return trace_impl<ANY>(m, sn, o, d, tmax, t_out, u_out, v_out);
}

// fp32 fast mode: the same traversal with the triangle test in fp32 on fp32
// copies of the records (half the bytes, twice the arithmetic rate).  Paths
// may then branch differently from the fp64 parity mode; the fraction of
// affected pixels is measured (tests/test_gpu_mesh.py) and reported.
constexpr float kTMin32 = 1e-5f;

struct Tri32 {
  float4 a, b, c;
};
__device__ __forceinline__ Tri32 load_tri32(const float4* __restrict__ r) {
  return Tri32{__ldg(r), __ldg(r + 1), __ldg(r + 2)};
}
__device__ __forceinline__ bool tri_test32(const Tri32& T, const float o[3], const float d[3],
                                           float& t, float& u, float& v) {
  const float4 a = T.a, b = T.b, c = T.c;
  const float v0[3] = {a.x, a.y, a.z}, e1[3] = {a.w, b.x, b.y}, e2[3] = {b.z, b.w, c.x};
  const float p[3] = {d[1] * e2[2] - d[2] * e2[1], d[2] * e2[0] - d[0] * e2[2],
                      d[0] * e2[1] - d[1] * e2[0]};
  const float det = (e1[0] * p[0] + e1[1] * p[1]) + e1[2] * p[2];
  if (det == 0.0f) return false;
  const float inv = 1.0f / det;
  const float s[3] = {o[0] - v0[0], o[1] - v0[1], o[2] - v0[2]};
  const float uu = ((s[0] * p[0] + s[1] * p[1]) + s[2] * p[2]) * inv;
  if (uu < 0.0f || uu > 1.0f) return false;
  const float q[3] = {s[1] * e1[2] - s[2] * e1[1], s[2] * e1[0] - s[0] * e1[2],
                      s[0] * e1[1] - s[1] * e1[0]};
  const float vv = ((d[0] * q[0] + d[1] * q[1]) + d[2] * q[2]) * inv;
  if (vv < 0.0f || uu + vv > 1.0f) return false;
  const float tt = ((e2[0] * q[0] + e2[1] * q[1]) + e2[2] * q[2]) * inv;
  if (!(tt > kTMin32)) return false;
  t = tt;
  u = uu;
  v = vv;
  return true;
}
__device__ __forceinline__ bool tri_hit32(const float4* __restrict__ r, const float o[3],
                                          const float d[3], float& t, float& u, float& v) {
  return tri_test32(load_tri32(r), o, d, t, u, v);
}

// SSTK: stack in shared memory laid out [entry][thread] (kSmemStackT
// entries of a kMThreads-thread CTA at smem_stack; see trace32_persistent);
// QN: quantised 64-byte nodes (m.nodesq).  Same hits in every form.
constexpr int kSmemStackT = 48;
template <bool ANY, bool SSTK = false, bool QN = false>
__device__ __forceinline__ int trace32_impl(const MeshDev& m, const float4* sn, const double o[3],
                                            const double d[3], double tmax, double& t_out,
                                            double& u_out, double& v_out,
                                            int* smem_stack = nullptr) {
  float of[3], df[3], inv[3], ooi[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    of[k] = float(o[k]);
    df[k] = float(d[k]);
    inv[k] = 1.0f / (fabsf(df[k]) > 1e-20f ? df[k] : copysignf(1e-20f, df[k]));
    ooi[k] = of[k] * inv[k];
  }
  int lstack[SSTK ? 1 : kStackDepth];
  int* const sstack = SSTK ? smem_stack + threadIdx.x : nullptr;
  auto push = [&](int sp, int val) {
    if constexpr (SSTK)
      sstack[sp * kMThreads] = val;
    else
      lstack[sp] = val;
  };
  auto top = [&](int sp) {
    if constexpr (SSTK)
      return sstack[sp * kMThreads];
    else
      return lstack[sp];
  };
  int sp = 0, node = 0;
  const float tmaxf = float(tmax);
  float best = tmaxf, bu = 0.0f, bv = 0.0f;
  int bslot = -1, bid = INT_MAX;
  for (;;) {
    if (node < 0) {
      // triangles two at a time: both records are requested before the
      // first test, so a two-triangle leaf costs one memory latency, not
      // two (tests and their order unchanged)
      const int first = (~node) >> 3, end = first + ((~node) & 7);
      for (int s0 = first; s0 < end; s0 += 2) {
        Tri32 tr[2];
        tr[0] = load_tri32(m.tri32 + 3 * size_t(s0));
        if (s0 + 1 < end) tr[1] = load_tri32(m.tri32 + 3 * size_t(s0 + 1));
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int sidx = s0 + e;
          if (sidx >= end) break;
          float t, u, v;
          if (!tri_test32(tr[e], of, df, t, u, v) || !(t <= best)) continue;
          if (ANY) {
            if (t < tmaxf) return sidx;
            continue;
          }
          const int id = __ldg(&m.orig[sidx]);
          if (t < best || id < bid) {
            best = t;
            bu = u;
            bv = v;
            bslot = sidx;
            bid = id;
          }
        }
      }
    } else {
      MG_DCHECK(node < m.nnodes && sp + 4 <= (SSTK ? kSmemStackT : kStackDepth));
      float tk[4];
      int ck[4];
      if constexpr (QN) {  // trace32_persistent's decode of the quantised node
        const float4* src = m.nodesq + size_t(kNodeQF4) * node;
        const float4 hd = __ldg(src), q0 = __ldg(src + 1), q1 = __ldg(src + 2), rf = __ldg(src + 3);
        const unsigned eb = __float_as_uint(hd.w);
        const float pa[3] = {hd.x, hd.y, hd.z};
        float A[3], Bo[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          A[a] = __uint_as_float(((eb >> (8 * a)) & 255u) << 23) * inv[a];
          Bo[a] = (pa[a] - of[a]) * inv[a];
        }
        const unsigned qw[6] = {__float_as_uint(q0.x), __float_as_uint(q0.y),
                                __float_as_uint(q0.z), __float_as_uint(q0.w),
                                __float_as_uint(q1.x), __float_as_uint(q1.y)};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float t[6];
#pragma unroll
          for (int f = 0; f < 6; ++f) {
            const float qf =
                __uint_as_float(__byte_perm(qw[f], 0x4B000000u, 0x7650u | unsigned(c))) -
                8388608.0f;
            t[f] = fmaf(qf, A[f % 3], Bo[f % 3]);
          }
          const float tn = fmaxf(fmaxf(fminf(t[0], t[3]), fminf(t[1], t[4])),
                                 fmaxf(fminf(t[2], t[5]), 0.0f));
          const float tf = fminf(fminf(fmaxf(t[0], t[3]), fmaxf(t[1], t[4])),
                                 fminf(fmaxf(t[2], t[5]), best));
          tk[c] = tn <= tf ? tn : INFINITY;
          ck[c] = __float_as_int(f4c(rf, c));
        }
      } else {
        const NodeW n = load_node<!SSTK>(m, sn, node);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float tc;
          const bool h = slab6(f4c(n.lx, c), f4c(n.ly, c), f4c(n.lz, c), f4c(n.hx, c),
                               f4c(n.hy, c), f4c(n.hz, c), ooi, inv, best, tc);
          tk[c] = h ? tc : INFINITY;
          ck[c] = __float_as_int(f4c(n.ref, c));
        }
      }
      auto cx = [&](int a, int b) {
        if (tk[b] < tk[a]) {
          const float tt = tk[a];
          tk[a] = tk[b];
          tk[b] = tt;
          const int cc = ck[a];
          ck[a] = ck[b];
          ck[b] = cc;
        }
      };
      if (!ANY || MG_ANY_SORT) {  // any-hit rays need no front-to-back order
        cx(0, 1);
        cx(2, 3);
        cx(0, 2);
        cx(1, 3);
        cx(1, 2);
      }
      if (ANY && !MG_ANY_SORT) {
        int nx = 0;
        bool have = false;
#pragma unroll
        for (int c = 3; c >= 0; --c) {
          if (tk[c] == INFINITY) continue;
          if (have) push(sp++, nx);
          nx = ck[c];
          have = true;
        }
        if (have) {
          node = nx;
          continue;
        }
      } else if (tk[0] != INFINITY) {
        if (tk[3] != INFINITY) push(sp++, ck[3]);
        if (tk[2] != INFINITY) push(sp++, ck[2]);
        if (tk[1] != INFINITY) push(sp++, ck[1]);
        node = ck[0];
        continue;
      }
    }
    if (sp == 0) break;
    node = top(--sp);
  }
  t_out = bslot < 0 ? INFINITY : double(best);
  u_out = double(bu);
  v_out = double(bv);
  return bslot;
}

// fp32 traversal as a persistent warp loop (Aila & Laine, "Understanding
// the efficiency of ray traversal on GPUs", HPG 2009: while-while with
// speculative traversal and replacement of terminated rays).  Each lane
// runs rays fetched from a queue counter in warp-aggregated batches; a lane
// whose ray terminates takes a new one at the top of the loop, so lanes of
// a warp do not idle until the warp's slowest ray is done.  Within a ray,
// inner nodes are traversed until every active lane holds a leaf (a lane
// that meets a leaf postpones it and keeps descending), then leaves are
// intersected together — fewer divergent inner/leaf iterations.  Same
// node / triangle tests and the same closest-hit rule (t, then the lower
// original index: independent of the visiting order) as trace32_impl, so
// the hits are identical.
//   fetch(i, o, d, tmax) -> id: loads queue entry i, returns the ray's id
//   finish(id, slot, t, u, v): writes the result (slot -1: no hit)
constexpr int kDone = INT_MAX;

// Traversal stack of the persistent loop.  Local memory interleaves a
// thread's entries with its warp-mates' at the same index, so lanes at
// different depths touch a different 128-byte row each (ncu: 1.8 of 32
// bytes used per local sector).  SMEM_STACK keeps the stack in shared
// memory laid out [entry][thread] instead: every lane hits its own bank at
// any depth.  kSmemStack entries (24 KB per 128-thread CTA) hold any BVH4 of
// depth <= kSmemStackMaxDepth (3 pushes per level); deeper scenes use the
// local-memory form.
constexpr int kSmemStack = 48;
constexpr int kSmemStackMaxDepth = (kSmemStack - 1) / 3 - 1;

template <bool ANY, bool SMEM_STACK = false, bool QNODES = false, class Fetch, class Finish>
__device__ __forceinline__ void trace32_persistent(const MeshDev& m, const float4* sn, int n,
                                                   unsigned int* counter, Fetch fetch,
                                                   Finish finish, int* smem_stack = nullptr) {
  const int lane = int(threadIdx.x & 31);
  int rid = -1;
  bool done = false;
  float of[3], df[3], inv[3], ooi[3];
  float tmaxf = 0.0f, best = 0.0f, bu = 0.0f, bv = 0.0f;
  int bslot = -1, bid = INT_MAX, node = kDone, leaf = 0, sp = 0;
  int lstack[SMEM_STACK ? 1 : kStackDepth];
  int* const sstack = SMEM_STACK ? smem_stack + threadIdx.x : nullptr;
  auto push = [&](int v) {
    MG_DCHECK(sp < (SMEM_STACK ? kSmemStack : kStackDepth));
    if constexpr (SMEM_STACK)
      sstack[(sp++) * kMThreads] = v;
    else
      lstack[sp++] = v;
  };
  auto pop = [&]() {
    if (sp == 0) return kDone;
    if constexpr (SMEM_STACK)
      return sstack[(--sp) * kMThreads];
    else
      return lstack[--sp];
  };
  for (;;) {
    const bool need = rid < 0 && !done;
    const unsigned needm = __ballot_sync(0xffffffffu, need);
    if (needm) {
      const int leader = __ffs(needm) - 1;
      unsigned base = 0;
      if (lane == leader) base = atomicAdd(counter, unsigned(__popc(needm)));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (need) {
        const int idx = int(base + unsigned(__popc(needm & ((1u << lane) - 1u))));
        if (idx < n) {
          double o[3], d[3], tm;
          rid = fetch(idx, o, d, tm);
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            of[k] = float(o[k]);
            df[k] = float(d[k]);
            inv[k] = 1.0f / (fabsf(df[k]) > 1e-20f ? df[k] : copysignf(1e-20f, df[k]));
            ooi[k] = of[k] * inv[k];
          }
          tmaxf = float(tm);
          best = tmaxf;
          bu = bv = 0.0f;
          bslot = -1;
          bid = INT_MAX;
          node = 0;
          leaf = 0;
          sp = 0;
        } else {
          done = true;
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (rid < 0) continue;
    // inner nodes until every active lane has a leaf waiting
    while (node >= 0 && node != kDone) {
      float tk[4];
      int ck[4];
      if constexpr (QNODES) {
        // 64-byte node: header, 24 plane bytes, refs.  Plane t of child c,
        // axis a: (p + q s - o) inv = q (s inv) + (p - o) inv, q decoded
        // exactly from its byte (0x4B0000qq as a float is 2^23 + q)
        const float4* src = m.nodesq + size_t(kNodeQF4) * node;
        const float4 hd = __ldg(src), q0 = __ldg(src + 1), q1 = __ldg(src + 2), rf = __ldg(src + 3);
        const unsigned eb = __float_as_uint(hd.w);
        const float pa[3] = {hd.x, hd.y, hd.z};
        float A[3], Bo[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          A[a] = __uint_as_float(((eb >> (8 * a)) & 255u) << 23) * inv[a];
          Bo[a] = (pa[a] - of[a]) * inv[a];
        }
        const unsigned qw[6] = {__float_as_uint(q0.x), __float_as_uint(q0.y),
                                __float_as_uint(q0.z), __float_as_uint(q0.w),
                                __float_as_uint(q1.x), __float_as_uint(q1.y)};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float t[6];
#pragma unroll
          for (int f = 0; f < 6; ++f) {
            const float qf =
                __uint_as_float(__byte_perm(qw[f], 0x4B000000u, 0x7650u | unsigned(c))) -
                8388608.0f;
            t[f] = fmaf(qf, A[f % 3], Bo[f % 3]);
          }
          const float tn = fmaxf(fmaxf(fminf(t[0], t[3]), fminf(t[1], t[4])),
                                 fmaxf(fminf(t[2], t[5]), 0.0f));
          const float tf = fminf(fminf(fmaxf(t[0], t[3]), fmaxf(t[1], t[4])),
                                 fminf(fmaxf(t[2], t[5]), best));
          tk[c] = tn <= tf ? tn : INFINITY;
          ck[c] = __float_as_int(f4c(rf, c));
        }
      } else {
        const NodeW nd = load_node<!SMEM_STACK>(m, sn, node);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float tc;
          const bool h = slab6(f4c(nd.lx, c), f4c(nd.ly, c), f4c(nd.lz, c), f4c(nd.hx, c),
                               f4c(nd.hy, c), f4c(nd.hz, c), ooi, inv, best, tc);
          tk[c] = h ? tc : INFINITY;
          ck[c] = __float_as_int(f4c(nd.ref, c));
        }
      }
      auto cx = [&](int a, int b) {
        if (tk[b] < tk[a]) {
          const float tt = tk[a];
          tk[a] = tk[b];
          tk[b] = tt;
          const int cc = ck[a];
          ck[a] = ck[b];
          ck[b] = cc;
        }
      };
      if (!ANY) {
        cx(0, 1);
        cx(2, 3);
        cx(0, 2);
        cx(1, 3);
        cx(1, 2);
        if (tk[0] != INFINITY) {
          if (tk[3] != INFINITY) push(ck[3]);
          if (tk[2] != INFINITY) push(ck[2]);
          if (tk[1] != INFINITY) push(ck[1]);
          node = ck[0];
        } else {
          node = pop();
        }
      } else {
        int nx = 0;
        bool have = false;
#pragma unroll
        for (int c = 3; c >= 0; --c) {
          if (tk[c] == INFINITY) continue;
          if (have) push(nx);
          nx = ck[c];
          have = true;
        }
        node = have ? nx : pop();
      }
      if (node < 0 && leaf == 0) {  // postpone the leaf, keep descending
        leaf = node;
        node = pop();
      }
      if (!__any_sync(__activemask(), leaf == 0)) break;
    }
    // the waiting leaves (and any leaf met next) of this lane
    bool hit_any = false;
    while (leaf < 0) {
      const int first = (~leaf) >> 3, end = first + ((~leaf) & 7);
      for (int s0 = first; s0 < end && !hit_any; s0 += 2) {
        Tri32 tr[2];
        tr[0] = load_tri32(m.tri32 + 3 * size_t(s0));
        if (s0 + 1 < end) tr[1] = load_tri32(m.tri32 + 3 * size_t(s0 + 1));
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int sidx = s0 + e;
          if (sidx >= end) break;
          float t, u, v;
          if (!tri_test32(tr[e], of, df, t, u, v) || !(t <= best)) continue;
          if (ANY) {
            if (t < tmaxf) {
              bslot = sidx;
              hit_any = true;
              break;
            }
            continue;
          }
          const int id = __ldg(&m.orig[sidx]);
          if (t < best || id < bid) {
            best = t;
            bu = u;
            bv = v;
            bslot = sidx;
            bid = id;
          }
        }
      }
      if (hit_any) {
        leaf = 0;
        node = kDone;
        break;
      }
      leaf = 0;
      if (node < 0) {
        leaf = node;
        node = pop();
      }
    }
    if (node == kDone && leaf == 0) {
      finish(rid, bslot, bslot < 0 ? double(INFINITY) : double(best), double(bu), double(bv));
      rid = -1;
    }
  }
}

// ---------------------------------------------------------------- BVH8
// Eight-child nodes (224 B, SoA: lo.x[8] lo.y[8] lo.z[8] hi.x[8] hi.y[8]
// hi.z[8] ref[8]; fp32 boxes rounded outwards and padded exactly like the
// BVH4 ones; empty slots: inverted box and ref ~0, an empty leaf) built from
// the same binary tree by opening the largest child until eight.  Half the
// levels of the BVH4: fewer dependent node fetches per ray, eight boxes
// tested per fetch.  Used by the fp32 persistent traversal only.
constexpr int kNode8F4 = 14;
constexpr int kSmemNodes8 = 64;  // top BVH8 nodes staged in shared memory (14 KB)

__device__ __forceinline__ void stage_nodes8(const MeshDev& m, float4* sn) {
  const int n = kNode8F4 * (m.nnodes8 < kSmemNodes8 ? m.nnodes8 : kSmemNodes8);
  for (int i = threadIdx.x; i < n; i += blockDim.x) sn[i] = m.nodes8[i];
  __syncthreads();
}

// half h (children 4h..4h+3) of node i: lx ly lz hx hy hz ref as float4s
struct Node8Half {
  float4 lx, ly, lz, hx, hy, hz, ref;
};
__device__ __forceinline__ Node8Half load_node8_half(const MeshDev& m, const float4* sn, int i,
                                                     int h) {
  const bool shared = i < kSmemNodes8;
  const float4* src = (shared ? sn : m.nodes8) + size_t(kNode8F4) * i + h;
  Node8Half n;
  if (shared) {
    n.lx = src[0];
    n.ly = src[2];
    n.lz = src[4];
    n.hx = src[6];
    n.hy = src[8];
    n.hz = src[10];
    n.ref = src[12];
  } else {
    n.lx = __ldg(src);
    n.ly = __ldg(src + 2);
    n.lz = __ldg(src + 4);
    n.hx = __ldg(src + 6);
    n.hy = __ldg(src + 8);
    n.hz = __ldg(src + 10);
    n.ref = __ldg(src + 12);
  }
  return n;
}

template <bool ANY, class Fetch, class Finish>
__device__ __forceinline__ void trace32_persistent8(const MeshDev& m, const float4* sn, int n,
                                                    unsigned int* counter, Fetch fetch,
                                                    Finish finish) {
  const int lane = int(threadIdx.x & 31);
  int rid = -1;
  bool done = false;
  float of[3], df[3], inv[3], ooi[3];
  float tmaxf = 0.0f, best = 0.0f, bu = 0.0f, bv = 0.0f;
  int bslot = -1, bid = INT_MAX, node = kDone, leaf = 0, sp = 0;
  int stack[kStackDepth];
  float stackt[kStackDepth];  // entry distance of each pushed child (culled when popped)
  Node8Half nh;
  auto pop = [&]() {
    while (sp > 0) {
      --sp;
      if (ANY || stackt[sp] <= best) return stack[sp];
    }
    return kDone;
  };
  for (;;) {
    const bool need = rid < 0 && !done;
    const unsigned needm = __ballot_sync(0xffffffffu, need);
    if (needm) {
      const int leader = __ffs(needm) - 1;
      unsigned base = 0;
      if (lane == leader) base = atomicAdd(counter, unsigned(__popc(needm)));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (need) {
        const int idx = int(base + unsigned(__popc(needm & ((1u << lane) - 1u))));
        if (idx < n) {
          double o[3], d[3], tm;
          rid = fetch(idx, o, d, tm);
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            of[k] = float(o[k]);
            df[k] = float(d[k]);
            inv[k] = 1.0f / (fabsf(df[k]) > 1e-20f ? df[k] : copysignf(1e-20f, df[k]));
            ooi[k] = of[k] * inv[k];
          }
          tmaxf = float(tm);
          best = tmaxf;
          bu = bv = 0.0f;
          bslot = -1;
          bid = INT_MAX;
          node = 0;
          leaf = 0;
          sp = 0;
        } else {
          done = true;
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (rid < 0) continue;
    while (node >= 0 && node != kDone) {
      // nearest hit child goes next, the other hits are pushed with their
      // entry distances; the node is read in two halves of four children
      int nx = kDone;
      float tn = INFINITY;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if ((c & 3) == 0) nh = load_node8_half(m, sn, node, c >> 2);
        float tc;
        if (!slab6(f4c(nh.lx, c & 3), f4c(nh.ly, c & 3), f4c(nh.lz, c & 3), f4c(nh.hx, c & 3),
                   f4c(nh.hy, c & 3), f4c(nh.hz, c & 3), ooi, inv, best, tc))
          continue;
        const int cr = __float_as_int(f4c(nh.ref, c & 3));
        if (ANY || tc < tn) {
          if (nx != kDone) {
            MG_DCHECK(sp < kStackDepth);
            stack[sp] = nx;
            stackt[sp] = tn;
            ++sp;
          }
          nx = cr;
          tn = tc;
        } else {
          MG_DCHECK(sp < kStackDepth);
          stack[sp] = cr;
          stackt[sp] = tc;
          ++sp;
        }
      }
      node = nx != kDone ? nx : pop();
      if (node < 0 && leaf == 0) {  // postpone the leaf, keep descending
        leaf = node;
        node = pop();
      }
      if (!__any_sync(__activemask(), leaf == 0)) break;
    }
    bool hit_any = false;
    while (leaf < 0) {
      const int first = (~leaf) >> 3, end = first + ((~leaf) & 7);
      for (int s0 = first; s0 < end && !hit_any; s0 += 2) {
        Tri32 tr[2];
        tr[0] = load_tri32(m.tri32 + 3 * size_t(s0));
        if (s0 + 1 < end) tr[1] = load_tri32(m.tri32 + 3 * size_t(s0 + 1));
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int sidx = s0 + e;
          if (sidx >= end) break;
          float t, u, v;
          if (!tri_test32(tr[e], of, df, t, u, v) || !(t <= best)) continue;
          if (ANY) {
            if (t < tmaxf) {
              bslot = sidx;
              hit_any = true;
              break;
            }
            continue;
          }
          const int id = __ldg(&m.orig[sidx]);
          if (t < best || id < bid) {
            best = t;
            bu = u;
            bv = v;
            bslot = sidx;
            bid = id;
          }
        }
      }
      if (hit_any) {
        leaf = 0;
        node = kDone;
        break;
      }
      leaf = 0;
      if (node < 0) {
        leaf = node;
        node = pop();
      }
    }
    if (node == kDone && leaf == 0) {
      finish(rid, bslot, bslot < 0 ? double(INFINITY) : double(best), double(bu), double(bv));
      rid = -1;
    }
  }
}

// traversal in the precision of the mode: fp64 (parity) or fp32 (fast)
template <bool ANY, class T>
__device__ __forceinline__ int trace_mode(const MeshDev& m, const float4* sn, const double o[3],
                                          const double d[3], double tmax, double& t_out,
                                          double& u_out, double& v_out) {
  if constexpr (sizeof(T) == 4)
    return trace32_impl<ANY>(m, sn, o, d, tmax, t_out, u_out, v_out);
  else
    return trace_impl<ANY>(m, sn, o, d, tmax, t_out, u_out, v_out);
}

template <bool ANY, class T>
__device__ __noinline__ int trace_t(const MeshDev& m, const float4* sn, const double o[3],
                                    const double d[3], double tmax, double& t_out, double& u_out,
                                    double& v_out) {
  return trace_mode<ANY, T>(m, sn, o, d, tmax, t_out, u_out, v_out);
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

__device__ __forceinline__ unsigned long long fixq(double v) {
  return (unsigned long long)llrint(v * kFixM);
}

// adjoint of a stored path, set s, channel weights w (oracle ms_scatter)
__device__ __forceinline__ void stage_nodes(const MeshDev& m, float4* sn) {
  const int n = kNodeF4 * (m.nnodes < kSmemNodes ? m.nnodes : kSmemNodes);
  for (int i = threadIdx.x; i < n; i += blockDim.x) sn[i] = m.nodes[i];
  __syncthreads();
}

// shared-memory arrays every tracing kernel declares
#define MESH_SMEM                       \
  __shared__ float4 sn[kNodeF4 * kSmemNodes]; \
  stage_nodes(m, sn)


inline MeshDev dev_of(const mg_mesh_scene* s) {
  MeshDev m;
  m.tri = s->tri;
  m.tri32 = s->tri32;
  m.orig = s->orig;
  m.obj = s->obj;
  m.nodes = s->nodes;
  m.nnodes = s->nnodes;
  m.nodes8 = s->nodes8;
  m.nnodes8 = s->nnodes8;
  m.nodesq = s->nodesq;
  return m;
}

inline MeshK make_k(const mg_mesh_scene* s, int W, int H, const double* view, uint64_t key,
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
  q.it_offset = nullptr;
  return q;
}

inline int check_view(const double* view) {
  if (!view) return fail(MG_EINVAL, "mesh scene: null view");
  const int maxv = int(view[24]);
  if (maxv < 1 || maxv > kMaxV) return fail(MG_EINVAL, "mesh scene: max_vertices must lie in [1, 8]");
  return MG_OK;
}

// megakernel sample pair (configs[3] form), mesh_megakernel.cu
int megakernel_pair(mg_ctx* ctx, mg_mesh_scene* s, const MeshK& q, int32_t dtype,
                    const void* target_img, const void* now, const void* prev,
                    unsigned long long* acc, long long np, double* loss_out);

}  // namespace mesh
}  // namespace mg
