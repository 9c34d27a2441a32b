// Host side of the mesh renderer: binned-SAH BVH build (32 bins on each axis, at most
// g_bvh_leaf triangles per leaf), breadth-first relabelling of the internal
// nodes so the top levels form one block every CTA stages in shared memory,
// 128-byte four-child nodes (the binary tree collapsed by opening the
// largest child first) with fp32 boxes rounded outwards and padded (the
// fp32 slab test never culls a triangle the fp64 test would hit); scene
// create / destroy / info.  DESIGN.md §12.
#include <algorithm>
#include <vector>

#include "mesh.cuh"

namespace mg {
bool g_mesh_megakernel = false;
int g_mesh_persistent = -1;
int g_mesh_tail = -1;
bool g_mesh_scatter_agg = false;
bool g_mesh_bvh8 = false;
bool g_mesh_smem_stack = true;
bool g_mesh_qnodes = true;
int g_bvh_axes = 3;
int g_bvh_bins = 32;
int g_bvh_leaf = 2;
namespace mesh {
namespace {

float f4c_host(const float4& v, int c) { return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w)); }

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
    // binned SAH over every axis with extent (g_bvh_axes = 1: the longest
    // centroid axis only, the round-1 builder)
    int mid = -1;
    {
      constexpr int kMaxBins = 64;
      const int kBins = g_bvh_bins;
      double best = INFINITY;
      int best_split = -1, best_axis = -1;
      auto bin_of = [&](int t, int ax) {
        const double ext = chi[ax] - clo[ax];
        int q = int(((cen[size_t(3 * t + ax)] - clo[ax]) / ext) * kBins);
        return q < 0 ? 0 : (q >= kBins ? kBins - 1 : q);
      };
      for (int ax = 0; ax < 3; ++ax) {
        if (g_bvh_axes == 1 && ax != axis) continue;
        if (!(chi[ax] - clo[ax] > 0.0)) continue;
        int cnt[kMaxBins] = {0};
        double bl[kMaxBins][3], bh[kMaxBins][3];
        for (int i = 0; i < kBins; ++i)
          for (int k = 0; k < 3; ++k) {
            bl[i][k] = INFINITY;
            bh[i][k] = -INFINITY;
          }
        for (int i = b; i < e; ++i) {
          const int t = idx[size_t(i)], q = bin_of(t, ax);
          cnt[q]++;
          for (int k = 0; k < 3; ++k) {
            bl[q][k] = std::min(bl[q][k], blo[size_t(3 * t + k)]);
            bh[q][k] = std::max(bh[q][k], bhi[size_t(3 * t + k)]);
          }
        }
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
            best_axis = ax;
          }
        }
      }
      if (best_split > 0) {
        auto it = std::partition(idx.begin() + b, idx.begin() + e, [&](int t) {
          return bin_of(t, best_axis) < best_split;
        });
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

}  // namespace
}  // namespace mesh
}  // namespace mg

using namespace mg;
using namespace mg::mesh;

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
  // Collapse the binary tree into 4-wide nodes (each BVH2 internal node
  // that becomes a BVH4 node adopts up to four descendants: repeatedly open
  // the child with the largest surface area), labelled breadth-first so the
  // top levels become nodes [0, kSmemNodes) for the shared-memory stage.
  const double diag = sqrt((shi[0] - slo[0]) * (shi[0] - slo[0]) +
                           (shi[1] - slo[1]) * (shi[1] - slo[1]) +
                           (shi[2] - slo[2]) * (shi[2] - slo[2]));
  const float pad = float(1e-5 * diag + 1e-7);
  auto sarea = [&](int c) {
    const TmpNode& nd = B.nodes[size_t(c)];
    return Builder::area(nd.lo, nd.hi);
  };
  auto wide_children = [&](int x) {
    std::vector<int> ch;
    const TmpNode& nd = B.nodes[size_t(x)];
    if (nd.left < 0) {  // a single-leaf tree: the root's only child
      ch.push_back(x);
      return ch;
    }
    ch = {nd.left, nd.right};
    while (ch.size() < 4) {
      int pick = -1;
      double best = -1.0;
      for (size_t k = 0; k < ch.size(); ++k)
        if (B.nodes[size_t(ch[k])].left >= 0 && sarea(ch[k]) > best) {
          best = sarea(ch[k]);
          pick = int(k);
        }
      if (pick < 0) break;
      const TmpNode& o = B.nodes[size_t(ch[size_t(pick)])];
      ch[size_t(pick)] = o.left;
      ch.push_back(o.right);
    }
    return ch;
  };
  std::vector<int> order;                 // BVH2 ids of the BVH4 nodes, BFS
  std::vector<std::vector<int>> kids;     // their children (BVH2 ids)
  std::vector<int> level;
  std::vector<int> label(B.nodes.size(), -1);
  order.push_back(0);
  label[0] = 0;
  level.push_back(0);
  int depth4 = 0;
  for (size_t h = 0; h < order.size(); ++h) {
    kids.push_back(wide_children(order[h]));
    for (int c : kids.back())
      if (B.nodes[size_t(c)].left >= 0 && c != order[h]) {
        label[size_t(c)] = int(order.size());
        order.push_back(c);
        level.push_back(level[h] + 1);
        depth4 = std::max(depth4, level[h] + 1);
      }
  }
  // each step pushes at most 3 children: the stack never exceeds 3 per level
  if (3 * (depth4 + 1) + 1 > kStackDepth)
    return fail(MG_EINVAL, "mg_meshscene_create: BVH deeper than the traversal stack");
  auto child_ref = [&](int c, int parent) {
    const TmpNode& nd = B.nodes[size_t(c)];
    return (nd.left >= 0 && c != parent) ? label[size_t(c)] : ~(nd.first * 8 + nd.count);
  };
  auto ibits = [](int v) {
    float f;
    memcpy(&f, &v, 4);
    return f;
  };
  const int nn = int(order.size());
  std::vector<float4> nodes(size_t(kNodeF4) * size_t(nn));
  for (int i = 0; i < nn; ++i) {
    float lo[3][4], hi[3][4];
    int ref[4];
    for (int c = 0; c < 4; ++c) {
      for (int a = 0; a < 3; ++a) {
        lo[a][c] = 1.0f;  // empty slot: inverted box
        hi[a][c] = -1.0f;
      }
      ref[c] = ~0;
    }
    const std::vector<int>& ch = kids[size_t(i)];
    for (size_t c = 0; c < ch.size(); ++c) {
      const TmpNode& nd = B.nodes[size_t(ch[c])];
      for (int a = 0; a < 3; ++a) {
        lo[a][c] = nextafterf(float(nd.lo[a]), -INFINITY) - pad;
        hi[a][c] = nextafterf(float(nd.hi[a]), INFINITY) + pad;
      }
      ref[c] = child_ref(ch[c], order[size_t(i)]);
    }
    float4* dst = &nodes[size_t(kNodeF4) * size_t(i)];
    dst[0] = make_float4(lo[0][0], lo[0][1], lo[0][2], lo[0][3]);
    dst[1] = make_float4(lo[1][0], lo[1][1], lo[1][2], lo[1][3]);
    dst[2] = make_float4(lo[2][0], lo[2][1], lo[2][2], lo[2][3]);
    dst[3] = make_float4(hi[0][0], hi[0][1], hi[0][2], hi[0][3]);
    dst[4] = make_float4(hi[1][0], hi[1][1], hi[1][2], hi[1][3]);
    dst[5] = make_float4(hi[2][0], hi[2][1], hi[2][2], hi[2][3]);
    dst[6] = make_float4(ibits(ref[0]), ibits(ref[1]), ibits(ref[2]), ibits(ref[3]));
    dst[7] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  }
  // Quantised copy of the BVH4 for the fp32 persistent traversal (64-byte
  // nodes): header (p.xyz = the node box's lower corner as the children's
  // float minimum, w = three biased exponents e: scale s = 2^(e-127) >=
  // extent / 255 per axis), then per axis and child one byte each for the
  // lower and upper plane, q_lo = floor((lo - p) / s), q_hi = ceil((hi - p)
  // / s) — exact in double, so the decoded box p + q s contains the padded
  // fp32 box (conservative like it); the child refs unchanged.  Empty slots
  // decode to the single point p (q = 0: hit with probability zero).
  std::vector<float4> nodesq(size_t(kNodeQF4) * size_t(nn));
  for (int i = 0; i < nn; ++i) {
    const float4* src = &nodes[size_t(kNodeF4) * size_t(i)];
    float lo[3][4], hi[3][4];
    bool used[4];
    for (int c = 0; c < 4; ++c) {
      for (int a = 0; a < 3; ++a) {
        lo[a][c] = f4c_host(src[a], c);
        hi[a][c] = f4c_host(src[3 + a], c);
      }
      used[c] = lo[0][c] <= hi[0][c];
    }
    float P[3];
    unsigned ex[3];
    double sc[3];
    for (int a = 0; a < 3; ++a) {
      float mn = INFINITY, mx = -INFINITY;
      for (int c = 0; c < 4; ++c)
        if (used[c]) {
          mn = std::min(mn, lo[a][c]);
          mx = std::max(mx, hi[a][c]);
        }
      if (!(mn <= mx)) mn = mx = 0.0f;  // no child (cannot happen for a built node)
      P[a] = mn;
      const double ext = double(mx) - double(mn);
      int e = -126;
      while (e < 127 && std::ldexp(255.0, e) < ext) ++e;
      ex[a] = unsigned(e + 127);
      sc[a] = std::ldexp(1.0, e);
    }
    unsigned q[6] = {0, 0, 0, 0, 0, 0};  // lo x, y, z, hi x, y, z (byte c = child c)
    for (int c = 0; c < 4; ++c) {
      if (!used[c]) continue;
      for (int a = 0; a < 3; ++a) {
        double ql = std::floor((double(lo[a][c]) - double(P[a])) / sc[a]);
        double qh = std::ceil((double(hi[a][c]) - double(P[a])) / sc[a]);
        ql = std::min(255.0, std::max(0.0, ql));
        qh = std::min(255.0, std::max(0.0, qh));
        q[a] |= unsigned(ql) << (8 * c);
        q[3 + a] |= unsigned(qh) << (8 * c);
      }
    }
    float4* dst = &nodesq[size_t(kNodeQF4) * size_t(i)];
    auto ubits = [](unsigned v) {
      float f;
      memcpy(&f, &v, 4);
      return f;
    };
    dst[0] = make_float4(P[0], P[1], P[2], ubits(ex[0] | (ex[1] << 8) | (ex[2] << 16)));
    dst[1] = make_float4(ubits(q[0]), ubits(q[1]), ubits(q[2]), ubits(q[3]));
    dst[2] = make_float4(ubits(q[4]), ubits(q[5]), 0.0f, 0.0f);
    dst[3] = src[6];
  }
  // The BVH8 of the fp32 persistent traversal: the same binary tree
  // collapsed eight-wide (open the largest-area internal child until eight
  // children), breadth-first labels, boxes rounded and padded as above.
  auto wide_children8 = [&](int x) {
    std::vector<int> ch;
    const TmpNode& nd = B.nodes[size_t(x)];
    if (nd.left < 0) {
      ch.push_back(x);
      return ch;
    }
    ch = {nd.left, nd.right};
    while (ch.size() < 8) {
      int pick = -1;
      double best = -1.0;
      for (size_t k = 0; k < ch.size(); ++k)
        if (B.nodes[size_t(ch[k])].left >= 0 && sarea(ch[k]) > best) {
          best = sarea(ch[k]);
          pick = int(k);
        }
      if (pick < 0) break;
      const TmpNode& o = B.nodes[size_t(ch[size_t(pick)])];
      ch[size_t(pick)] = o.left;
      ch.push_back(o.right);
    }
    return ch;
  };
  std::vector<int> order8{0}, level8{0};
  std::vector<std::vector<int>> kids8;
  std::vector<int> label8(B.nodes.size(), -1);
  label8[0] = 0;
  int depth8 = 0;
  for (size_t h = 0; h < order8.size(); ++h) {
    kids8.push_back(wide_children8(order8[h]));
    for (int c : kids8.back())
      if (B.nodes[size_t(c)].left >= 0 && c != order8[h]) {
        label8[size_t(c)] = int(order8.size());
        order8.push_back(c);
        level8.push_back(level8[h] + 1);
        depth8 = std::max(depth8, level8[h] + 1);
      }
  }
  // each step pushes at most 7 children
  // (the optional eight-wide traversal needs 7 pushes per level: a scene too
  // deep for its stack keeps the four-wide traversal, depth8 = -1)
  const bool bvh8_ok = 7 * (depth8 + 1) + 1 <= kStackDepth;
  const int nn8 = int(order8.size());
  std::vector<float4> nodes8(size_t(kNode8F4) * size_t(nn8));
  for (int i = 0; i < nn8; ++i) {
    float f[7][8];
    for (int c = 0; c < 8; ++c) {
      for (int a = 0; a < 3; ++a) {
        f[a][c] = 1.0f;  // empty slot: inverted box, empty leaf
        f[3 + a][c] = -1.0f;
      }
      f[6][c] = ibits(~0);
    }
    const std::vector<int>& ch = kids8[size_t(i)];
    for (size_t c = 0; c < ch.size(); ++c) {
      const TmpNode& nd = B.nodes[size_t(ch[c])];
      for (int a = 0; a < 3; ++a) {
        f[a][c] = nextafterf(float(nd.lo[a]), -INFINITY) - pad;
        f[3 + a][c] = nextafterf(float(nd.hi[a]), INFINITY) + pad;
      }
      const int ref = (nd.left >= 0 && ch[c] != order8[size_t(i)])
                          ? label8[size_t(ch[c])]
                          : ~(nd.first * 8 + nd.count);
      f[6][c] = ibits(ref);
    }
    float4* dst = &nodes8[size_t(kNode8F4) * size_t(i)];
    for (int fl = 0; fl < 7; ++fl)
      for (int hlf = 0; hlf < 2; ++hlf)
        dst[2 * fl + hlf] = make_float4(f[fl][4 * hlf], f[fl][4 * hlf + 1], f[fl][4 * hlf + 2],
                                        f[fl][4 * hlf + 3]);
  }
  std::vector<double> stri(kRec * T);
  std::vector<int> sorig(T), sobj(T);
  std::vector<float4> stri32(3 * T);
  for (size_t s = 0; s < T; ++s) {
    const int k = B.idx[s];
    memcpy(&stri[kRec * s], tri + kRec * size_t(k), sizeof(double) * kRec);
    sorig[s] = k;
    sobj[s] = obj[k];
    const double* r = tri + kRec * size_t(k);
    stri32[3 * s] = make_float4(float(r[0]), float(r[1]), float(r[2]), float(r[3]));
    stri32[3 * s + 1] = make_float4(float(r[4]), float(r[5]), float(r[6]), float(r[7]));
    stri32[3 * s + 2] = make_float4(float(r[8]), 0.0f, 0.0f, 0.0f);
  }
  mg_mesh_scene* sc = new mg_mesh_scene();
  sc->T = tri_count;
  sc->nobj = nobj;
  sc->nch = channels;
  sc->R = tex_res;
  sc->nnodes = nn;
  sc->depth = depth4;
  sc->nnodes8 = nn8;
  sc->depth8 = bvh8_ok ? depth8 : -1;
  cudaError_t e = cudaMalloc(&sc->tri, sizeof(double) * stri.size());
  if (e == cudaSuccess) e = cudaMalloc(&sc->tri32, sizeof(float4) * stri32.size());
  if (e == cudaSuccess)
    e = cudaMemcpy(sc->tri32, stri32.data(), sizeof(float4) * stri32.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&sc->orig, sizeof(int) * T);
  if (e == cudaSuccess) e = cudaMalloc(&sc->obj, sizeof(int) * T);
  if (e == cudaSuccess) e = cudaMalloc(&sc->nodes, sizeof(float4) * nodes.size());
  if (e == cudaSuccess) e = cudaMalloc(&sc->nodesq, sizeof(float4) * nodesq.size());
  if (e == cudaSuccess)
    e = cudaMemcpy(sc->nodesq, nodesq.data(), sizeof(float4) * nodesq.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&sc->nodes8, sizeof(float4) * nodes8.size());
  if (e == cudaSuccess)
    e = cudaMemcpy(sc->nodes8, nodes8.data(), sizeof(float4) * nodes8.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&sc->work, sizeof(unsigned int));
  if (e == cudaSuccess)
    e = cudaMemcpy(sc->tri, stri.data(), sizeof(double) * stri.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(sc->orig, sorig.data(), sizeof(int) * T, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(sc->obj, sobj.data(), sizeof(int) * T, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(sc->nodes, nodes.data(), sizeof(float4) * nodes.size(), cudaMemcpyHostToDevice);
  // pageable copies may return before the DMA lands; later kernels run on
  // non-blocking context streams, so fence once here
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaFree(sc->tri);
    cudaFree(sc->tri32);
    cudaFree(sc->orig);
    cudaFree(sc->obj);
    cudaFree(sc->nodes);
    cudaFree(sc->nodes8);
    cudaFree(sc->nodesq);
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
  cudaFree(s->tri32);
  cudaFree(s->orig);
  cudaFree(s->obj);
  cudaFree(s->nodes);
  cudaFree(s->nodes8);
  cudaFree(s->nodesq);
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

}  // extern "C"
