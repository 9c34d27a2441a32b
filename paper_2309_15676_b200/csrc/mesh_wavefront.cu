// Mesh renderer, wavefront form (the default for configs[3] and [4]):
// SoA path state, per-depth isect / shade / shadow stages over compacted
// queues, per-pixel adjoint scatter; bit-identical to the megakernel and the
// oracle.  DESIGN.md §12.
#include <type_traits>
#include "mesh.cuh"

namespace mg {
namespace mesh {
namespace {

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
  // record layout (sparse depths): [base, validity, set 0, set 1], a set =
  // [A C dSn | invfb dSb] = 11 slots
  static constexpr int stride = 24;
  __host__ __device__ static constexpr int slot(int f) {
    return 2 + (f < 6    ? (f / 3) * 11 + f % 3
                : f < 8  ? (f - 6) * 11 + 6
                : f < 14 ? ((f - 8) / 3) * 11 + 7 + (f - 8) % 3
                : f < 16 ? (f - 14) * 11 + 10
                         : ((f - 16) / 3) * 11 + 3 + (f - 16) % 3);
  }
};
template <>
struct VF<5> {
  static constexpr int n = 54, A = 0, invfb = 6, C = 12, dfn = 18, dfb = 36;
  // record layout (sparse depths): [base, validity, set 0, set 1], a set =
  // [A C dfn | invfb dfb] = 27 slots
  static constexpr int stride = 56;
  __host__ __device__ static constexpr int slot(int f) {
    return 2 + (f < 6    ? (f / 3) * 27 + f % 3
                : f < 12 ? ((f - 6) / 3) * 27 + 15 + (f - 6) % 3
                : f < 18 ? ((f - 12) / 3) * 27 + 3 + (f - 12) % 3
                : f < 36 ? ((f - 18) / 9) * 27 + 6 + (f - 18) % 9
                         : ((f - 36) / 9) * 27 + 18 + (f - 36) % 9);
  }
};

// every field has a slot of its own behind the two header slots
template <int NCH>
constexpr bool vf_slots_ok() {
  bool used[VF<NCH>::stride] = {};
  for (int f = 0; f < VF<NCH>::n; ++f) {
    const int k = VF<NCH>::slot(f);
    if (k < 2 || k >= VF<NCH>::stride || used[k]) return false;
    used[k] = true;
  }
  return true;
}
static_assert(vf_slots_ok<4>() && vf_slots_ok<5>(), "vertex record layout");

template <class T>
struct WF {
  double *ox, *oy, *oz, *dx, *dy, *dz;       // [P] ray
  double *ht, *hu, *hv;                       // [P] hit
  double *sox, *soy, *soz, *sdx, *sdy, *sdz, *stm;  // [P] shadow ray
  T *beta, *L, *E, *pendC;                    // [6][P]
  int *nv, *hslot, *q0, *q1, *sq;             // [P]
  int* vbase;                                 // [kMaxV][PS]
  // [kMaxV][PS]: the vertex's NEE (vnee) / bounce (vbnc) fields are valid;
  // invalid fields are never read (the scatter substitutes zeros), so they
  // need not be written
  unsigned char *vnee, *vbnc;
  // depths < vf_rec_from<NCH>(): [v][field][PS] planes (every path alive: coalesced);
  // depths >= vf_rec_from<NCH>(): [v][PS][stride] records (few survivors: a path's fields
  // share 4-7 sectors instead of one sector per field)
  T* vdat;
  // [4][kMaxV + 1]: queue counts, shadow-queue counts, and the fetch
  // counters of the persistent isect / shadow traversals
  unsigned int* cnt;
  int P, PS, npix, pix0, nprop, nvf;
};


template <class T>
size_t wf_bytes(int npix, int nprop, int nvf) {
  const size_t P = size_t(npix) * (nprop + 1), PS = size_t(npix) * nprop;
  return sizeof(double) * 16 * P + sizeof(T) * 24 * P + sizeof(int) * 5 * P +
         sizeof(int) * kMaxV * PS + sizeof(T) * kMaxV * nvf * PS + 2 * kMaxV * PS +
         sizeof(unsigned int) * 4 * (kMaxV + 1) + 256 * 40;
}

// Texel-major copies of the two parameter sets for the shade stage: texel
// (obj, t) at cell obj*R2 + t holds its NCH channels in TS slots (padded to
// one 16/32-byte aligned group), so a path vertex gathers its texel with one
// or two vector loads from one sector instead of NCH sectors a plane apart.
template <class T, int NCH>
struct TexIlv {
  static constexpr int TS = NCH == 4 ? 4 : 8;
};

// planar [obj][ch][R2] -> texel-major [cell][TS]: a CTA reads 256 cells
// channel by channel (coalesced), transposes through shared memory and
// stores the 256 x TS block with 16-byte vector stores.
template <class T, int NCH>
__global__ void __launch_bounds__(256) tex_ilv_kernel(int cells, int R2, const T* __restrict__ th,
                                                      T* __restrict__ out) {
  constexpr int TS = TexIlv<T, NCH>::TS;
  constexpr int VW = 16 / sizeof(T);  // elements per 16-byte store
  __shared__ __align__(16) T sm[256 * TS];
  for (int c0 = blockIdx.x * 256; c0 < cells; c0 += gridDim.x * 256) {
    const int k = c0 + threadIdx.x;
    if (k < cells) {
      const int obj = k / R2, tex = k - obj * R2;
#pragma unroll
      for (int c = 0; c < TS; ++c)
        sm[threadIdx.x * TS + c] = c < NCH ? th[(size_t(obj) * NCH + c) * R2 + tex] : T(0);
    }
    __syncthreads();
    const int nv = (cells - c0 < 256 ? cells - c0 : 256) * TS / VW;
    const uint4* src = reinterpret_cast<const uint4*>(sm);
    uint4* dst = reinterpret_cast<uint4*>(out + size_t(c0) * TS);
#pragma unroll
    for (int u = 0; u < TS * 256 / VW / 256; ++u) {
      const int j = threadIdx.x + u * 256;
      if (j < nv) dst[j] = src[j];
    }
    __syncthreads();
  }
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
  w.vnee = (unsigned char*)take(kMaxV * size_t(w.PS));
  w.vbnc = (unsigned char*)take(kMaxV * size_t(w.PS));
  w.vdat = (T*)take(sizeof(T) * kMaxV * size_t(nvf) * size_t(w.PS));
  w.cnt = (unsigned int*)take(sizeof(unsigned int) * 4 * (kMaxV + 1));
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
// (callers check the slot against their queue's capacity with MG_DCHECK)

// Depths >= vf_rec_from<NCH>() (0-based) store records, the others planes.
// The choice is a compile-time property of every access (REC): as a
// run-time branch in the accessors it cost configs[4] 0.9 ms per iteration.
// 5 channels (224-byte records): planes at depth 0, where every path is
// alive (configs[4] 7.21 ms against 7.61 with records everywhere);
// 4 channels (96-byte records): records everywhere (configs[3] 0.87 ms
// against 0.895).  Build switch for A/B: MG_VF_REC_FROM = 0 records
// everywhere, 99 planes everywhere, d records from depth d.
#ifndef MG_VF_REC_FROM
#define MG_VF_REC_FROM -1
#endif
template <int NCH>
__host__ __device__ constexpr int vf_rec_from() {
  return MG_VF_REC_FROM >= 0 ? MG_VF_REC_FROM : (NCH == 4 ? 0 : 1);
}
// vertex header: the texel's parameter base and the NEE / bounce validity
// bytes; at record depths they live in the record's first two slots
// (slot 0: base, slot 1: validity bytes 0 and 1)
template <bool REC, class T>
__device__ __forceinline__ int& vh_base(const WF<T>& w, int v, int p) {
  static_assert(sizeof(T) >= 4, "header slots");
  if constexpr (REC)
    return *reinterpret_cast<int*>(&w.vdat[(size_t(v) * w.PS + p) * w.nvf]);
  else
    return w.vbase[size_t(v) * w.PS + p];
}
template <bool REC, class T>
__device__ __forceinline__ unsigned char& vh_nee(const WF<T>& w, int v, int p) {
  if constexpr (REC)
    return reinterpret_cast<unsigned char*>(&w.vdat[(size_t(v) * w.PS + p) * w.nvf + 1])[0];
  else
    return w.vnee[size_t(v) * w.PS + p];
}
template <bool REC, class T>
__device__ __forceinline__ unsigned char& vh_bnc(const WF<T>& w, int v, int p) {
  if constexpr (REC)
    return reinterpret_cast<unsigned char*>(&w.vdat[(size_t(v) * w.PS + p) * w.nvf + 1])[1];
  else
    return w.vbnc[size_t(v) * w.PS + p];
}
// the shadow stages clear one validity byte: layout picked at run time
template <int NCH, class T>
__device__ __forceinline__ void vh_nee_clear(const WF<T>& w, int v, int p) {
  if (v >= vf_rec_from<NCH>())
    vh_nee<true>(w, v, p) = 0;
  else
    vh_nee<false>(w, v, p) = 0;
}
template <int NCH, bool REC, class T>
__device__ __forceinline__ T& vf(const WF<T>& w, int v, int f, int p) {
  using F = VF<NCH>;
  if constexpr (REC)
    return w.vdat[(size_t(v) * w.PS + p) * F::stride + F::slot(f)];
  else
    return w.vdat[(size_t(v) * F::stride + f) * size_t(w.PS) + p];
}

template <class T>
__global__ void __launch_bounds__(kMThreads) wf_gen_kernel(MeshK q, WF<T> w) {
  if (q.it_offset) q.iteration += __ldg(q.it_offset);
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
    const int slot = trace_mode<false, T>(m, sn, o, d, INFINITY, t, bu, bv);
    w.hslot[p] = slot;
    w.ht[p] = t;
    w.hu[p] = bu;
    w.hv[p] = bv;
  }
}

// fp32 mode, BVH8: the persistent traversals over the eight-wide tree
// (kP8Blocks CTAs of 128 per SM: 85 registers hold a node's 56 box / ref
// words without spilling)
#ifndef MG_P8_BLOCKS
#define MG_P8_BLOCKS 6
#endif
constexpr int kP8Blocks = MG_P8_BLOCKS;
__global__ void __launch_bounds__(kMThreads, kP8Blocks) wf_isect_p8_kernel(MeshDev m, WF<float> w, int v) {
  __shared__ float4 sn[kNode8F4 * kSmemNodes8];
  stage_nodes8(m, sn);
  const int n = int(w.cnt[v]);
  const int* qin = (v & 1) ? w.q1 : w.q0;
  trace32_persistent8<false>(
      m, sn, n, &w.cnt[2 * (kMaxV + 1) + v],
      [&](int i, double o[3], double d[3], double& tm) {
        const int p = qin[i];
        o[0] = w.ox[p];
        o[1] = w.oy[p];
        o[2] = w.oz[p];
        d[0] = w.dx[p];
        d[1] = w.dy[p];
        d[2] = w.dz[p];
        tm = INFINITY;
        return p;
      },
      [&](int p, int slot, double t, double u, double vv) {
        w.hslot[p] = slot;
        w.ht[p] = t;
        w.hu[p] = u;
        w.hv[p] = vv;
      });
}

// fp32 mode: persistent closest-hit traversal (trace32_persistent)
// SSTK: traversal stack in shared memory (24 KB per CTA; the top-node
// stage is then off)
template <bool SSTK, bool QN = false>
__global__ void __launch_bounds__(kMThreads, 8) wf_isect_p_kernel(MeshDev m, WF<float> w, int v) {
  __shared__ float4 sn[SSTK ? 1 : kNodeF4 * kSmemNodes];
  __shared__ int sstk[SSTK ? kSmemStack * kMThreads : 1];
  if (!SSTK) stage_nodes(m, sn);
  const int n = int(w.cnt[v]);
  const int* qin = (v & 1) ? w.q1 : w.q0;
  trace32_persistent<false, SSTK, QN>(
      m, sn, n, &w.cnt[2 * (kMaxV + 1) + v],
      [&](int i, double o[3], double d[3], double& tm) {
        const int p = qin[i];
        o[0] = w.ox[p];
        o[1] = w.oy[p];
        o[2] = w.oz[p];
        d[0] = w.dx[p];
        d[1] = w.dy[p];
        d[2] = w.dz[p];
        tm = INFINITY;
        return p;
      },
      [&](int p, int slot, double t, double u, double vv) {
        w.hslot[p] = slot;
        w.ht[p] = t;
        w.hu[p] = u;
        w.hv[p] = vv;
      },
      sstk);
}

// One queued path's shade step at depth v: texel, NEE sample + shadow-ray
// set-up, the BSDF values of the evaluated parameter sets, the Malley bounce
// and the stored adjoint fields.  want_shadow / want_bounce: the path joins
// this depth's shadow queue / the next depth's queue.  Shared by
// wf_shade_kernel and wf_tail_kernel (identical per-path arithmetic).
// The path state one shade step consumes and produces.  The stage kernel
// loads / stores it around the call; the tail kernel keeps it in registers
// from one depth to the next.
template <class T>
struct PathIO {
  int slot;                  // in: hit triangle slot (< 0: escaped)
  double o[3], d[3];         // in: the ray
  double t, bu, bv;          // in: hit distance and barycentrics (slot >= 0)
  T beta[2][3];              // in: throughput of the evaluated sets; out (want_bounce): next depth's
  double so[3], sd[3], stm;  // out (want_shadow): the NEE ray
  T pendC[2][3];             // out (want_shadow): the NEE contribution if unoccluded
  double on[3], dn[3];       // out (want_bounce): the next ray
};

// parameter sets a path evaluates: path 0 (A) and the FD path at theta_t
// and theta_{t-1}; the other proportional paths at theta_t only
template <class T>
__device__ __forceinline__ int path_sets(const WF<T>& w, int p) {
  const int k = p / w.npix;
  return (k == 0 || k == w.nprop) ? 2 : 1;
}

// REGS: the outputs stay in io (tail kernel); otherwise each is stored to
// the path-state arrays as soon as it is computed (stage kernel: holding
// them to the end of the call cost 25 registers and a resident CTA).
template <class T, int NCH, bool REC, bool REGS>
__device__ __forceinline__ void shade_path(const MeshK& q, const MeshDev& m, const WF<T>& w, int v,
                                           int p, PathIO<T>& io, const T* __restrict__ th0,
                                           const T* __restrict__ th1, int maxv, int R2, double la,
                                           bool& want_shadow, bool& want_bounce) {
  const int slot = io.slot;
  constexpr int TS = TexIlv<T, NCH>::TS;  // th0 / th1: texel-major copies
  using F = VF<NCH>;
  const double* V = q.view;
  const T* th[2] = {th0, th1};
  const int k = p / w.npix, pix = w.pix0 + (p - k * w.npix);
  const bool store = p < w.PS;
  // parameter sets evaluated: path 0 (A) and the FD path at theta_t and
  // theta_{t-1}; the other proportional paths at theta_t only
  const int ns = (k == 0 || k == w.nprop) ? 2 : 1;
  T beta[2][3];
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      beta[s][c] = s < ns ? io.beta[s][c] : T(0);
  if (slot < 0) {  // escaped: environment
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (s >= ns) break;
        // L += E is left to the consumer (wf_scatter_kernel): the
        // escape is the path's last event, so (L + E) there is the same
        // sum, and the scattered read-modify-write of L is saved
        w.E[size_t(s * 3 + c) * w.P + p] = beta[s][c] * T(V[21 + c]);
      }
  } else {
    const double o[3] = {io.o[0], io.o[1], io.o[2]}, d[3] = {io.d[0], io.d[1], io.d[2]};
    const double t = io.t, bu = io.bu, bv = io.bv;
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
    const int oid = __ldg(&m.obj[slot]), tex = ty * q.R + tx;
    const int pbase = oid * NCH * R2 + tex;
    const size_t cell = size_t(oid) * R2 + tex;
    w.nv[p] = v + 1;
    if (store) vh_base<REC>(w, v, p) = pbase;
    bool nee_done = false, bounce_done = false;
    T base[2][3], rough[2], metal[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (s >= ns) {  // the set is not evaluated: no texel gathers
#pragma unroll
        for (int c = 0; c < 3; ++c) base[s][c] = T(0);
        rough[s] = metal[s] = T(0);
        continue;
      }
      T x[TS];
      const T* tp = th[s] + cell * TS;
      if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int g = 0; g < TS; g += 4) {
          const float4 f4 = __ldg(reinterpret_cast<const float4*>(tp + g));
          x[g] = f4.x;
          x[g + 1] = f4.y;
          x[g + 2] = f4.z;
          x[g + 3] = f4.w;
        }
      } else {
#pragma unroll
        for (int g = 0; g < (NCH + 1) / 2 * 2; g += 2) {
          const double2 d2 = __ldg(reinterpret_cast<const double2*>(tp + g));
          x[g] = d2.x;
          x[g + 1] = d2.y;
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) base[s][c] = x[c];
      rough[s] = x[3];
      metal[s] = NCH == 5 ? x[4] : T(0);
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
              for (int kk = 0; kk < 3; ++kk) vf<NCH, REC>(w, v, F::dfn + s * 9 + c * 3 + kk, p) = df[c][kk];
        } else {
          T dS;
          bsdf_m0<T>(base[s], rough[s], nT, wT, woT, f, dS);
          if (store) vf<NCH, REC>(w, v, VF<4>::dSn + s, p) = dS;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const T A = beta[s][c] * T(gl * V[18 + c]);
          const T Cc = A * f[c];
          if (store) {
            vf<NCH, REC>(w, v, F::A + s * 3 + c, p) = A;
            vf<NCH, REC>(w, v, F::C + s * 3 + c, p) = Cc;
          }
          if constexpr (REGS)
            io.pendC[s][c] = Cc;
          else
            w.pendC[size_t(s * 3 + c) * w.P + p] = Cc;
        }
      }
      if constexpr (REGS) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          io.so[c] = xo[c];
          io.sd[c] = wl3[c];
        }
        io.stm = wl - kOff;
      } else {
        w.sox[p] = xo[0];
        w.soy[p] = xo[1];
        w.soz[p] = xo[2];
        w.sdx[p] = wl3[0];
        w.sdy[p] = wl3[1];
        w.sdz[p] = wl3[2];
        w.stm[p] = wl - kOff;
      }
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
                  vf<NCH, REC>(w, v, F::dfb + s * 9 + c * 3 + kk, p) = df[c][kk];
          } else {
            T dS;
            bsdf_m0<T>(base[s], rough[s], nT, wiT, woT, f, dS);
            if (store) vf<NCH, REC>(w, v, VF<4>::dSb + s, p) = dS;
          }
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            if (store) vf<NCH, REC>(w, v, F::invfb + s * 3 + c, p) = f[c] != T(0) ? T(1) / f[c] : T(0);
            if constexpr (REGS)
              io.beta[s][c] = beta[s][c] * (f[c] * T(kPiM));
            else
              w.beta[size_t(s * 3 + c) * w.P + p] = beta[s][c] * (f[c] * T(kPiM));
          }
        }
        if constexpr (REGS) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            io.on[c] = xo[c];
            io.dn[c] = wi[c];
          }
        } else {
          w.ox[p] = xo[0];
          w.oy[p] = xo[1];
          w.oz[p] = xo[2];
          w.dx[p] = wi[0];
          w.dy[p] = wi[1];
          w.dz[p] = wi[2];
        }
        want_bounce = true;
      }
    }
    if (store) {
      vh_nee<REC>(w, v, p) = nee_done;
      vh_bnc<REC>(w, v, p) = bounce_done;
    }
  }
}

// fp32: 4 CTAs/SM (128 registers, no spills)
#ifndef MG_SHADE_BLOCKS
#define MG_SHADE_BLOCKS 4
#endif
template <class T, int NCH, bool REC>
__global__ void __launch_bounds__(kMThreads, sizeof(T) == 4 ? MG_SHADE_BLOCKS : 1)
    wf_shade_kernel(MeshK q, MeshDev m, WF<T> w, int v, const T* __restrict__ th0,
                    const T* __restrict__ th1) {
  if (q.it_offset) q.iteration += __ldg(q.it_offset);
  const double* V = q.view;
  const int maxv = int(V[24]);
  const int R2 = q.R * q.R;
  const int n = int(w.cnt[v]);
  const int* qin = (v & 1) ? w.q1 : w.q0;
  int* qout = (v & 1) ? w.q0 : w.q1;
  const double la = (V[15] - V[14]) * (V[17] - V[16]);
  // software pipeline: the next queue entry and its hit slot are requested
  // (and the hit triangle's record prefetched into L2) one iteration ahead,
  // so the dependent chain queue -> path -> slot -> triangle of an
  // iteration overlaps the previous iteration's shading
#ifndef MG_SHADE_PIPE
#define MG_SHADE_PIPE 1
#endif
  const int stride = gridDim.x * kMThreads;
  int i = blockIdx.x * kMThreads + threadIdx.x;
  int pn = -1, slotn = -1;
  auto fetch = [&](int j) {
    pn = -1;
    slotn = -1;
    if (j < n) {
      pn = qin[j];
      slotn = w.hslot[pn];
      if (slotn >= 0) {
        const char* r = reinterpret_cast<const char*>(m.tri + size_t(kRec) * slotn);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(r));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(r + 128));
      }
    }
  };
  if (MG_SHADE_PIPE) fetch(i);
  for (; i - int(threadIdx.x) < n; i += stride) {
    bool want_shadow = false, want_bounce = false;
    int p = -1;
    int slot = -1;
    if (MG_SHADE_PIPE) {
      p = pn;
      slot = slotn;
      fetch(i + stride);
    } else if (i < n) {
      p = qin[i];
      slot = w.hslot[p];
    }
    if (p >= 0) {
      PathIO<T> io;
      io.slot = slot;
      const int ns = path_sets(w, p);
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          io.beta[s][c] = s < ns ? w.beta[size_t(s * 3 + c) * w.P + p] : T(0);
      if (slot >= 0) {
        io.o[0] = w.ox[p];
        io.o[1] = w.oy[p];
        io.o[2] = w.oz[p];
        io.d[0] = w.dx[p];
        io.d[1] = w.dy[p];
        io.d[2] = w.dz[p];
        io.t = w.ht[p];
        io.bu = w.hu[p];
        io.bv = w.hv[p];
      }
      shade_path<T, NCH, REC, false>(q, m, w, v, p, io, th0, th1, maxv, R2, la, want_shadow,
                                     want_bounce);
    }
    const int qs = enqueue(want_shadow, &w.cnt[kMaxV + 1 + v]);
    MG_DCHECK(qs < w.P);
    if (qs >= 0) w.sq[qs] = p;
    const int qb = enqueue(want_bounce, &w.cnt[v + 1]);
    MG_DCHECK(qb < w.P);
    if (qb >= 0) qout[qb] = p;
  }
}

template <class T, int NCH>
__global__ void __launch_bounds__(kMThreads, 8) wf_shadow_kernel(MeshDev m, WF<T> w, int v) {
  MESH_SMEM;
  const int n = int(w.cnt[kMaxV + 1 + v]);
  for (int i = blockIdx.x * kMThreads + threadIdx.x; i < n; i += gridDim.x * kMThreads) {
    const int p = w.sq[i];
    const double o[3] = {w.sox[p], w.soy[p], w.soz[p]}, d[3] = {w.sdx[p], w.sdy[p], w.sdz[p]};
    double ts, tu, tv;
    if (trace_mode<true, T>(m, sn, o, d, w.stm[p], ts, tu, tv) < 0) {
      const int k = p / w.npix;
      const int nj = (k == 0 || k == w.nprop) ? 6 : 3;
      for (int j = 0; j < nj; ++j) w.L[size_t(j) * w.P + p] += w.pendC[size_t(j) * w.P + p];
    } else if (p < w.PS) {  // occluded: no NEE data at this vertex
      vh_nee_clear<NCH>(w, v, p);
    }
  }
}

// fp32 mode: persistent any-hit traversal of the NEE rays
template <int NCH, bool SSTK, bool QN = false>
__global__ void __launch_bounds__(kMThreads, 8) wf_shadow_p_kernel(MeshDev m, WF<float> w, int v) {
  __shared__ float4 sn[SSTK ? 1 : kNodeF4 * kSmemNodes];
  __shared__ int sstk[SSTK ? kSmemStack * kMThreads : 1];
  if (!SSTK) stage_nodes(m, sn);
  const int n = int(w.cnt[kMaxV + 1 + v]);
  trace32_persistent<true, SSTK, QN>(
      m, sn, n, &w.cnt[3 * (kMaxV + 1) + v],
      [&](int i, double o[3], double d[3], double& tm) {
        const int p = w.sq[i];
        o[0] = w.sox[p];
        o[1] = w.soy[p];
        o[2] = w.soz[p];
        d[0] = w.sdx[p];
        d[1] = w.sdy[p];
        d[2] = w.sdz[p];
        tm = w.stm[p];
        return p;
      },
      [&](int p, int slot, double, double, double) {
        if (slot < 0) {
          const int k = p / w.npix;
          const int nj = (k == 0 || k == w.nprop) ? 6 : 3;
          for (int j = 0; j < nj; ++j) w.L[size_t(j) * w.P + p] += w.pendC[size_t(j) * w.P + p];
        } else if (p < w.PS) {  // occluded: no NEE data at this vertex
          vh_nee_clear<NCH>(w, v, p);
        }
      },
      sstk);
}

template <int NCH>
__global__ void __launch_bounds__(kMThreads, kP8Blocks) wf_shadow_p8_kernel(MeshDev m, WF<float> w, int v) {
  __shared__ float4 sn[kNode8F4 * kSmemNodes8];
  stage_nodes8(m, sn);
  const int n = int(w.cnt[kMaxV + 1 + v]);
  trace32_persistent8<true>(
      m, sn, n, &w.cnt[3 * (kMaxV + 1) + v],
      [&](int i, double o[3], double d[3], double& tm) {
        const int p = w.sq[i];
        o[0] = w.sox[p];
        o[1] = w.soy[p];
        o[2] = w.soz[p];
        d[0] = w.sdx[p];
        d[1] = w.sdy[p];
        d[2] = w.sdz[p];
        tm = w.stm[p];
        return p;
      },
      [&](int p, int slot, double, double, double) {
        if (slot < 0) {
          const int k = p / w.npix;
          const int nj = (k == 0 || k == w.nprop) ? 6 : 3;
          for (int j = 0; j < nj; ++j) w.L[size_t(j) * w.P + p] += w.pendC[size_t(j) * w.P + p];
        } else if (p < w.PS) {  // occluded: no NEE data at this vertex
          vh_nee_clear<NCH>(w, v, p);
        }
      });
}

// Tail of the wavefront (fp32 mode).  After a few depths the queues are
// small (configs[4]: 5.2M paths enter depth 1, 0.69M depth 3, 75k depth 8)
// and every stage launch is bounded by its slowest ray, not by throughput:
// the depth-8 shadow stage takes 0.11 ms for 24k rays.  From depth v0 on,
// one launch carries each remaining path through all its remaining depths —
// closest hit, shade_path, any-hit NEE ray, next bounce — so the long
// traversals of different depths overlap instead of each stage waiting for
// its slowest ray.  Lanes whose path ends take the next queue entry
// (warp-aggregated fetch at the top of every depth step).  The per-path
// arithmetic is the wavefront's (same traversal results: closest hit by t,
// then the lower original index; any-hit is a visibility test), so the
// result is bit-identical.
// SSTK / QN: the traversal stack in shared memory, quantised nodes (as the
// persistent stages).
// CTAs per SM: 4 (128 registers) for 5 channels, 3 (168) for 4 channels
// (configs[3] 0.895 -> 0.867 ms; configs[4] 7.22 -> 7.33 ms with 3)
#ifndef MG_TAIL_BLOCKS
#define MG_TAIL_BLOCKS -1
#endif
template <int NCH>
__host__ __device__ constexpr int tail_blocks() {
  return MG_TAIL_BLOCKS > 0 ? MG_TAIL_BLOCKS : (NCH == 4 ? 3 : 4);
}
template <int NCH, bool SSTK, bool QN>
__global__ void __launch_bounds__(kMThreads, tail_blocks<NCH>())
    wf_tail_kernel(MeshK q, MeshDev m, WF<float> w, int v0, const float* __restrict__ th0,
                   const float* __restrict__ th1) {
  __shared__ float4 sn[SSTK ? 1 : kNodeF4 * kSmemNodes];
  __shared__ int sstk[SSTK ? kSmemStackT * kMThreads : 1];
  if (!SSTK) stage_nodes(m, sn);
  if (q.it_offset) q.iteration += __ldg(q.it_offset);
  const double* V = q.view;
  const int maxv = int(V[24]);
  const int R2 = q.R * q.R;
  const double la = (V[15] - V[14]) * (V[17] - V[16]);
  const int n = int(w.cnt[v0]);
  const int* qin = (v0 & 1) ? w.q1 : w.q0;
  // depth v0's isect fetch counter: that stage does not run
  unsigned int* fetch = &w.cnt[2 * (kMaxV + 1) + v0];
  const int lane = int(threadIdx.x & 31);
  int p = -1, v = v0;
  bool done = false;
  // the path's ray and throughput stay in registers from depth to depth
  // (and its hit, NEE ray and pending NEE term never reach memory): as
  // global arrays every depth step paid their write, an L2 round trip to
  // read them back and one sector per field
  PathIO<float> io;
  int ns = 1;
  for (;;) {
    const bool need = p < 0 && !done;
    const unsigned needm = __ballot_sync(0xffffffffu, need);
    if (needm) {
      const int leader = __ffs(needm) - 1;
      unsigned base = 0;
      if (lane == leader) base = atomicAdd(fetch, unsigned(__popc(needm)));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (need) {
        const int idx = int(base + unsigned(__popc(needm & ((1u << lane) - 1u))));
        if (idx < n) {
          p = qin[idx];
          v = v0;
          ns = path_sets(w, p);
          io.o[0] = w.ox[p];
          io.o[1] = w.oy[p];
          io.o[2] = w.oz[p];
          io.d[0] = w.dx[p];
          io.d[1] = w.dy[p];
          io.d[2] = w.dz[p];
#pragma unroll
          for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int c = 0; c < 3; ++c)
              io.beta[s][c] = s < ns ? w.beta[size_t(s * 3 + c) * w.P + p] : 0.0f;
        } else {
          done = true;
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (p < 0) continue;
    io.t = INFINITY;
    io.bu = 0.0;
    io.bv = 0.0;
    io.slot = trace32_impl<false, SSTK, QN>(m, sn, io.o, io.d, INFINITY, io.t, io.bu, io.bv, sstk);
    bool want_shadow = false, want_bounce = false;
    if (vf_rec_from<NCH>() <= 1 || v >= vf_rec_from<NCH>())  // the tail starts at depth >= 1
      shade_path<float, NCH, true, true>(q, m, w, v, p, io, th0, th1, maxv, R2, la, want_shadow,
                                   want_bounce);
    else
      shade_path<float, NCH, false, true>(q, m, w, v, p, io, th0, th1, maxv, R2, la, want_shadow,
                                    want_bounce);
    if (want_shadow) {
      double ts, tu, tv;
      if (trace32_impl<true, SSTK, QN>(m, sn, io.so, io.sd, io.stm, ts, tu, tv, sstk) < 0) {
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
          for (int c = 0; c < 3; ++c)
            if (s < ns) w.L[size_t(s * 3 + c) * w.P + p] += io.pendC[s][c];
      } else if (p < w.PS) {  // occluded: no NEE data at this vertex
        vh_nee_clear<NCH>(w, v, p);
      }
    }
    if (want_bounce) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        io.o[c] = io.on[c];
        io.d[c] = io.dn[c];
      }
      ++v;
    } else {
      p = -1;
    }
  }
}

// Where the fixed-point adjoints go.
//  * One rank (ilv = 1): one accumulator, texel-interleaved
//    [obj][texel][prop | diff][NCH] — the NCH channel atomics of a vertex
//    land in 1-2 adjacent 32-byte sectors instead of NCH sectors a plane
//    apart (the accumulator is larger than L2, so every sector touched is a
//    DRAM read-modify-write).  mesh_finalize_ilv transposes it back into the
//    planar parameter order [obj][ch][texel].
//  * Tile-sharded ranks (configs[3]/[4] over NVLink, ilv = 0): parameter j
//    (planar order) is owned by rank j / shard, whose accumulator
//    [2][shard] is reached through a peer pointer — the scatter IS the
//    reduce-scatter (integer atomics commute, so the owner's sums are
//    independent of the ranks' order).
constexpr int kMaxRanks = 8;
struct AccTable {
  unsigned long long* ptr[kMaxRanks];
  int shard;  // parameters per rank
  int ilv;    // 1: single texel-interleaved accumulator
  // ilv only, optional: one bit per texel cell, set with every vertex added
  // to the cell (mg_meshscene_set_touch_map; consumed and cleared by
  // mg_meta_update_fixed_touch)
  unsigned int* touch;
};

__device__ __forceinline__ unsigned long long* acc_slot(const AccTable& a, int j, int which) {
  const int r = j / a.shard;
  return a.ptr[r] + size_t(which) * a.shard + (j - r * a.shard);
}

// the accumulator cells of vertex parameter base `base` (= obj*NCH*R2 + texel)
template <int NCH, bool ILV>
struct AccCell {
  unsigned long long* q;  // ILV: the texel's [2][NCH] cell
  int base, R2;
  __device__ __forceinline__ AccCell(const AccTable& a, int b, int r2) : base(b), R2(r2) {
    if (ILV) {
      const int obj = b / (NCH * r2), tex = b - obj * NCH * r2;
      const size_t cell = size_t(obj) * r2 + tex;
      q = a.ptr[0] + cell * (2 * NCH);
      if (a.touch) atomicOr(&a.touch[cell >> 5], 1u << (cell & 31));
    }
  }
  __device__ __forceinline__ unsigned long long* at(const AccTable& a, int which, int k) const {
    MG_DCHECK(which >= 0 && which < 2 && k >= 0 && k < NCH && base >= 0);
    MG_DCHECK(ILV ? (q + which * NCH + k) < a.ptr[0] + 2 * size_t(a.shard)
                  : (base + k * R2) / a.shard < kMaxRanks);
    return ILV ? q + which * NCH + k : acc_slot(a, base + k * R2, which);
  }
};

// Adds val[k] (fixed point) to the NCH accumulator words of `cell`, set
// `which`.  agg: warp-aggregated — the converged lanes adding to the same
// cell (__match_any_sync on the parameter base) are summed first and one
// lane per cell issues the NCH atomics (integer sums: the same result in any
// order, so bit-identical to one atomic per lane).
template <int NCH, bool ILV>
__device__ __forceinline__ void cell_add(bool agg, const AccTable& acc,
                                         const AccCell<NCH, ILV>& cell, int which,
                                         const unsigned long long (&val)[NCH]) {
  if (!agg) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) red_add_u64(cell.at(acc, which, k), val[k]);
    return;
  }
  const unsigned act = __activemask();
  const unsigned peers = __match_any_sync(act, cell.base);
  const int lane = int(threadIdx.x & 31), leader = __ffs(peers) - 1;
  unsigned rem = lane == leader ? (peers & ~(1u << lane)) : 0u;
  unsigned long long sum[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) sum[k] = val[k];
  while (__any_sync(act, rem != 0u)) {
    const int src = rem ? __ffs(rem) - 1 : lane;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const unsigned long long y = __shfl_sync(act, val[k], src);
      if (rem) sum[k] += y;
    }
    rem &= rem - 1u;
  }
  if (lane == leader)
#pragma unroll
    for (int k = 0; k < NCH; ++k) red_add_u64(cell.at(acc, which, k), sum[k]);
}

// Per-vertex adjoint terms of stored path p, parameter set s (megakernel
// `scatter` / oracle ms_scatter), before the channel weights: X[c][0] for
// base colour c, X[c][1] roughness, X[c][2] metalness (NCH 5); Q is the
// suffix radiance.  combine() applies weights wt:
//   g[c] = wt[c] X[c][0],  g[3] = sum_c wt[c] X[c][1],  g[4] = sum_c wt[c] X[c][2].
template <class T, int NCH, bool REC>
__device__ __forceinline__ void vertex_terms(const WF<T>& w, int v, int p, int s, const T Q[3],
                                             bool ne, bool bn, T X[3][NCH - 2]) {
  using F = VF<NCH>;
  // fields of an absent NEE / bounce event read as +0 (what the megakernel
  // and the oracle store for them)
  auto fn = [&](int f) { return ne ? vf<NCH, REC>(w, v, f, p) : T(0); };
  auto fbn = [&](int f) { return bn ? vf<NCH, REC>(w, v, f, p) : T(0); };
  if constexpr (NCH == 5) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const T A = fn(F::A + s * 3 + c), fb = fbn(F::invfb + s * 3 + c);
      const int dn = F::dfn + s * 9 + c * 3, db = F::dfb + s * 9 + c * 3;
      X[c][0] = A * fn(dn) + Q[c] * (fb * fbn(db));
      X[c][2] = A * fn(dn + 1) + Q[c] * (fb * fbn(db + 1));
      X[c][1] = A * fn(dn + 2) + Q[c] * (fb * fbn(db + 2));
    }
  } else {
    const T dSn = fn(F::dSn + s), dSb = fbn(F::dSb + s);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const T A = fn(F::A + s * 3 + c), ifb = fbn(F::invfb + s * 3 + c);
      X[c][0] = (A / T(kPiM)) + Q[c] * (ifb / T(kPiM));
      X[c][1] = A * dSn + Q[c] * (ifb * dSb);
    }
  }
}

template <class T, int NCH>
__device__ __forceinline__ void combine(const T X[3][NCH - 2], const T wt[3], T g[NCH]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) g[c] = wt[c] * X[c][0];
#pragma unroll
  for (int k = 1; k < NCH - 2; ++k) {
    T a = T(0);
#pragma unroll
    for (int c = 0; c < 3; ++c) a += wt[c] * X[c][k];
    g[2 + k] = a;
  }
}

// The two walks are inlined into the scatter kernel: as out-of-line calls
// (ABI call, 416-byte stack frame, spilled arguments) configs[4] took
// 8.02 ms per iteration, inlined 7.77 ms (same 124 registers).
#ifndef MG_SCATTER_NOINLINE
#define MG_SCATTER_NOINLINE 0
#endif
#if MG_SCATTER_NOINLINE
#define MG_SCATTER_INLINE __device__ __noinline__
#else
#define MG_SCATTER_INLINE __device__ __forceinline__
#endif
// adjoint of stored proportional path p (set 0) into the prop accumulator
template <class T, int NCH, bool ILV>
MG_SCATTER_INLINE void wf_scatter(const WF<T>& w, int p, const T wt[3], int R2,
                                        const AccTable& acc, bool agg) {
  using F = VF<NCH>;
  T Q[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) Q[c] = w.E[size_t(c) * w.P + p];
  // the warp's lanes walk their vertices in lockstep by vertex index (lane
  // idle while v >= its own count): every field load of an iteration reads
  // one [v][field] plane, coalesced across the warp's neighbouring paths.
  // Walking each lane from its own last vertex put lanes of one iteration
  // in different planes (ncu: 57 % of the scatter's L2 sectors excessive).
  // Same per-lane operation order, same warp iteration count.
  const int nvp = w.nv[p];
#ifndef MG_SCATTER_LOCKSTEP
#define MG_SCATTER_LOCKSTEP 1
#endif
  const int vtop = MG_SCATTER_LOCKSTEP ? __reduce_max_sync(__activemask(), unsigned(nvp)) : nvp;
  auto vertex = [&](int v, auto rec) {
    constexpr bool REC = decltype(rec)::value;
    const AccCell<NCH, ILV> cell(acc, vh_base<REC>(w, v, p), R2);
    const bool ne = vh_nee<REC>(w, v, p), bn = vh_bnc<REC>(w, v, p);
    T X[3][NCH - 2], g[NCH];
    vertex_terms<T, NCH, REC>(w, v, p, 0, Q, ne, bn, X);
    combine<T, NCH>(X, wt, g);
    unsigned long long d[NCH];
#pragma unroll
    for (int k = 0; k < NCH; ++k) d[k] = fixq(double(g[k]));
    cell_add<NCH, ILV>(agg, acc, cell, 0, d);
#pragma unroll
    for (int c = 0; c < 3; ++c) Q[c] = Q[c] + (ne ? vf<NCH, REC>(w, v, F::C + c, p) : T(0));
  };
  // record depths, then plane depths: the layout is a compile-time
  // property of each loop
  int v = vtop - 1;
  for (; v >= vf_rec_from<NCH>(); --v)
    if (v < nvp) vertex(v, std::true_type{});
  for (; v >= 0; --v)
    if (v < nvp) vertex(v, std::false_type{});
}

// Path A (p = pixel i) in ONE walk: its proportional adjoint (set 0,
// weights wt) and both finite-difference adjoints (set 0 with wC0, set 1
// with wC1).  The two FD terms of a parameter are added as integers before
// the atomic — the same fixed-point sum as two separate atomics, bit for bit.
template <class T, int NCH, bool ILV>
MG_SCATTER_INLINE void wf_scatter_a(const WF<T>& w, int p, const T wt[3], const T wC0[3],
                                          const T wC1[3], int R2, const AccTable& acc,
                                          bool agg) {
  using F = VF<NCH>;
  T Q0[3], Q1[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    Q0[c] = w.E[size_t(c) * w.P + p];
    Q1[c] = w.E[size_t(3 + c) * w.P + p];
  }
  // the warp's lanes walk their vertices in lockstep by vertex index (lane
  // idle while v >= its own count): every field load of an iteration reads
  // one [v][field] plane, coalesced across the warp's neighbouring paths.
  // Walking each lane from its own last vertex put lanes of one iteration
  // in different planes (ncu: 57 % of the scatter's L2 sectors excessive).
  // Same per-lane operation order, same warp iteration count.
  const int nvp = w.nv[p];
#ifndef MG_SCATTER_LOCKSTEP
#define MG_SCATTER_LOCKSTEP 1
#endif
  const int vtop = MG_SCATTER_LOCKSTEP ? __reduce_max_sync(__activemask(), unsigned(nvp)) : nvp;
  auto vertex = [&](int v, auto rec) {
    constexpr bool REC = decltype(rec)::value;
    const AccCell<NCH, ILV> cell(acc, vh_base<REC>(w, v, p), R2);
    const bool ne = vh_nee<REC>(w, v, p), bn = vh_bnc<REC>(w, v, p);
    T X[3][NCH - 2], g[NCH];
    unsigned long long d[NCH];
    vertex_terms<T, NCH, REC>(w, v, p, 0, Q0, ne, bn, X);
    combine<T, NCH>(X, wt, g);
#pragma unroll
    for (int k = 0; k < NCH; ++k) d[k] = fixq(double(g[k]));
    cell_add<NCH, ILV>(agg, acc, cell, 0, d);
    combine<T, NCH>(X, wC0, g);
#pragma unroll
    for (int k = 0; k < NCH; ++k) d[k] = fixq(double(g[k]));
    vertex_terms<T, NCH, REC>(w, v, p, 1, Q1, ne, bn, X);
    combine<T, NCH>(X, wC1, g);
#pragma unroll
    for (int k = 0; k < NCH; ++k) d[k] = d[k] + fixq(double(g[k]));
    cell_add<NCH, ILV>(agg, acc, cell, 1, d);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      Q0[c] = Q0[c] + (ne ? vf<NCH, REC>(w, v, F::C + c, p) : T(0));
      Q1[c] = Q1[c] + (ne ? vf<NCH, REC>(w, v, F::C + 3 + c, p) : T(0));
    }
  };
  int v = vtop - 1;
  for (; v >= vf_rec_from<NCH>(); --v)
    if (v < nvp) vertex(v, std::true_type{});
  for (; v >= 0; --v)
    if (v < nvp) vertex(v, std::false_type{});
}

constexpr int kMaxProp = 8;

// 6 CTAs/SM (<= 80 registers).  With the per-vertex records the walk holds
// few values: configs[4] 7.05 -> 7.00 ms, configs[3] 0.866 -> 0.850 ms
// against 4 CTAs/SM (5: 7.01 / 0.851, 3: 7.19 / 0.883).  (With one plane
// per field, 4 had measured 2 % faster than the unconstrained 168-227
// registers and 6 / 8 slower or equal.)
#ifndef MG_SCATTER_BLOCKS
#define MG_SCATTER_BLOCKS 6
#endif
template <class T, int NCH, bool ILV>
__global__ void __launch_bounds__(kMThreads, MG_SCATTER_BLOCKS)
    wf_scatter_kernel(MeshK q, WF<T> w, const T* __restrict__ target_img, AccTable acc,
                      ReducePartials* partials, unsigned int* counter, double* loss_out,
                      bool agg) {
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
      auto rad = [&](int ch, int path) {  // path radiance L + E (escape term deferred)
        const size_t o = size_t(ch) * w.P + path;
        return w.L[o] + w.E[o];
      };
      for (int j = 0; j < n; ++j) r[j][c] = rad(c, j * w.npix + i) - Is;
      wC0[c] = T(2) * (rad(c, pc) - Is);
      wC1[c] = T(-2) * (rad(3 + c, pc) - Is);
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
      if (j == 0)
        wf_scatter_a<T, NCH, ILV>(w, i, wt, wC0, wC1, R2, acc, agg);
      else
        wf_scatter<T, NCH, ILV>(w, j * w.npix + i, wt, R2, acc, agg);
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

// texel-interleaved accumulator [cells = nobj*R2][2][NCH] -> planar prop /
// diff [obj][ch][texel]; accumulator zeroed.  A CTA takes 256 consecutive
// cells per step: the 256 x 2 x NCH words are copied to shared memory with
// 16-byte cp.async (double-buffered: the next tile is in flight while this
// one is written out), zeroed in global memory with coalesced 16-byte
// stores, then written one thread per cell (coalesced along the texel).
constexpr int kFinCells = 256;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = unsigned(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}

template <class T, int NCH>
__global__ void __launch_bounds__(kFinCells)
    mesh_finalize_ilv_kernel(long long cells, int R2, unsigned long long* __restrict__ acc,
                             T* __restrict__ prop, T* __restrict__ diff) {
  constexpr int kW = 2 * NCH;  // words per cell (even: tiles are 16-byte aligned)
  __shared__ __align__(16) long long sm[2][kFinCells * kW];
  const long long step = (long long)gridDim.x * kFinCells;
  auto issue = [&](long long c0, int b) {
    if (c0 < cells) {
      const int n2 = int(cells - c0 < kFinCells ? cells - c0 : kFinCells) * (kW / 2);
      const ulonglong2* a2 = reinterpret_cast<const ulonglong2*>(acc + c0 * kW);
#pragma unroll
      for (int u = 0; u < NCH; ++u) {
        const int j = threadIdx.x + u * kFinCells;
        if (j < n2) cp_async16(&sm[b][2 * j], a2 + j);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  int b = 0;
  long long c0 = blockIdx.x * (long long)kFinCells;
  issue(c0, 0);
  for (; c0 < cells; c0 += step, b ^= 1) {
    issue(c0 + step, b ^ 1);
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    const int nc = int(cells - c0 < kFinCells ? cells - c0 : kFinCells);
    ulonglong2* a2 = reinterpret_cast<ulonglong2*>(acc + c0 * kW);
#pragma unroll
    for (int u = 0; u < NCH; ++u) {  // this thread's own copies have landed
      const int j = threadIdx.x + u * kFinCells;
      if (j < nc * (kW / 2)) a2[j] = make_ulonglong2(0ull, 0ull);
    }
    __syncthreads();
    const int t = threadIdx.x;
    if (t < nc) {
      const long long k = c0 + t, obj = k / R2, tex = k - obj * R2;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const long long o = (obj * NCH + c) * R2 + tex;
        prop[o] = T(double(sm[b][t * kW + c]) / kFixM);
        diff[o] = T(double(sm[b][t * kW + NCH + c]) / kFixM);
      }
    }
    __syncthreads();  // buffer b is refilled by the next issue
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

template <class T>
int finalize_ilv(mg_ctx* ctx, int nch, long long cells, int R2, unsigned long long* acc, T* prop,
                 T* diff) {
  const int grid = grid_for(ctx, cells, kFinCells, 8);
  if (nch == 5)
    mesh_finalize_ilv_kernel<T, 5><<<grid, kFinCells, 0, ctx->stream>>>(cells, R2, acc, prop, diff);
  else
    mesh_finalize_ilv_kernel<T, 4><<<grid, kFinCells, 0, ctx->stream>>>(cells, R2, acc, prop, diff);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

}  // namespace

template <class T, int NCH>
int wavefront_pair(mg_ctx* ctx, mg_mesh_scene* s, const MeshK& q, int nprop, const T* target_img,
                   const T* now, const T* prev, const AccTable& acc, double* loss_out) {
  const int npix = q.W * (q.row1 - q.row0);
  if (npix == 0) {
    MG_CUDA_TRY(cudaMemsetAsync(loss_out, 0, sizeof(double), ctx->stream));
    return MG_OK;
  }
  if (int64_t(npix) * (nprop + 1) > 0x7fffffffLL) return fail(MG_EINVAL, "mesh scene: image too large");
  constexpr int TS = TexIlv<T, NCH>::TS;
  const long long cells = (long long)s->nobj * q.R * q.R;
  const size_t tex_bytes = (sizeof(T) * TS * size_t(cells) + 255) & ~size_t(255);
  // the two texel-copy slots come first: their addresses depend on the scene
  // only, not on the tile size, so a copy can outlive the call that made it
  const size_t need = 2 * tex_bytes + wf_bytes<T>(npix, nprop, VF<NCH>::stride);
  if (need > s->wf_cap) {
    MG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    cudaFree(s->wf);
    s->wf = nullptr;
    s->wf_cap = 0;
    s->last_now_slot = -1;
    MG_CUDA_TRY(cudaMalloc(&s->wf, need));
    s->wf_cap = need;
  }
  WF<T> w = wf_carve<T>(static_cast<char*>(s->wf) + 2 * tex_bytes, npix, nprop, VF<NCH>::stride);
  w.pix0 = q.row0 * q.W;
  T* slot[2];
  slot[0] = static_cast<T*>(s->wf);
  slot[1] = reinterpret_cast<T*>(static_cast<char*>(s->wf) + tex_bytes);
  T* thI[2];
  {
    const int dt = sizeof(T) == 8 ? MG_F64 : MG_F32;
    const bool reuse = s->prev_reuse && s->last_now_slot >= 0 && s->last_dtype == dt &&
                       prev == s->last_now && now != prev;
    const int sp = reuse ? s->last_now_slot : 1, sn = 1 - sp;
    const int tg = grid_for(ctx, cells, 256, 8);
    thI[0] = slot[sn];
    thI[1] = slot[sp];
    tex_ilv_kernel<T, NCH><<<tg, 256, 0, ctx->stream>>>(int(cells), q.R * q.R, now, thI[0]);
    if (!reuse)
      tex_ilv_kernel<T, NCH><<<tg, 256, 0, ctx->stream>>>(int(cells), q.R * q.R, prev, thI[1]);
    MG_LAUNCH_CHECK(ctx);
    s->last_now = now;
    s->last_now_slot = sn;
    s->last_dtype = dt;
  }
  const MeshDev m = dev_of(s);
  s->last_cnt = w.cnt;
  MG_CUDA_TRY(cudaMemsetAsync(w.cnt, 0, sizeof(unsigned int) * 4 * (kMaxV + 1), ctx->stream));
  const int grid = grid_for(ctx, w.P, kMThreads, 8);
  // persistent traversals: one resident wave (8 CTAs of 128 per SM; the
  // BVH8 kernels kP8Blocks)
  const int pgrid = grid;
  const int pgrid8 = grid_for(ctx, w.P, kMThreads, kP8Blocks);
  const bool sstk = g_mesh_smem_stack && s->depth <= kSmemStackMaxDepth;
  const int pmode = g_mesh_persistent >= 0 ? g_mesh_persistent : 3;
  wf_gen_kernel<T><<<grid, kMThreads, 0, ctx->stream>>>(q, w);
  MG_LAUNCH_CHECK(ctx);
  const int maxv = int(q.view[24]);
  static const char* kDepthName[kMaxV] = {"wavefront depth 0", "wavefront depth 1",
                                          "wavefront depth 2", "wavefront depth 3",
                                          "wavefront depth 4", "wavefront depth 5",
                                          "wavefront depth 6", "wavefront depth 7"};
  const int tail_from =
      g_mesh_tail >= 0 ? g_mesh_tail : (maxv - kMeshTailDepths > 1 ? maxv - kMeshTailDepths : 1);
  for (int v = 0; v < maxv; ++v) {
    MG_NVTX(kDepthName[v]);
    if constexpr (sizeof(T) == 4) {
      if (tail_from > 0 && v >= tail_from) {
        const int tgrid = grid_for(ctx, w.P, kMThreads, tail_blocks<NCH>());
        if (sstk && g_mesh_qnodes)
          wf_tail_kernel<NCH, true, true><<<tgrid, kMThreads, 0, ctx->stream>>>(q, m, w, v, thI[0],
                                                                                thI[1]);
        else
          wf_tail_kernel<NCH, false, false><<<tgrid, kMThreads, 0, ctx->stream>>>(q, m, w, v,
                                                                                  thI[0], thI[1]);
        MG_LAUNCH_CHECK(ctx);
        break;
      }
    }
    if constexpr (sizeof(T) == 4) {
      if ((pmode & 1) && g_mesh_bvh8 && s->depth8 >= 0)
        wf_isect_p8_kernel<<<pgrid8, kMThreads, 0, ctx->stream>>>(m, w, v);
      else if ((pmode & 1) && sstk && g_mesh_qnodes)
        wf_isect_p_kernel<true, true><<<pgrid, kMThreads, 0, ctx->stream>>>(m, w, v);
      else if ((pmode & 1) && sstk)
        wf_isect_p_kernel<true><<<pgrid, kMThreads, 0, ctx->stream>>>(m, w, v);
      else if (pmode & 1)
        wf_isect_p_kernel<false><<<pgrid, kMThreads, 0, ctx->stream>>>(m, w, v);
      else
        wf_isect_kernel<T><<<grid, kMThreads, 0, ctx->stream>>>(m, w, v);
    } else {
      wf_isect_kernel<T><<<grid, kMThreads, 0, ctx->stream>>>(m, w, v);
    }
    MG_LAUNCH_CHECK(ctx);
    if (v >= vf_rec_from<NCH>())
      wf_shade_kernel<T, NCH, true><<<grid, kMThreads, 0, ctx->stream>>>(q, m, w, v, thI[0],
                                                                        thI[1]);
    else
      wf_shade_kernel<T, NCH, false><<<grid, kMThreads, 0, ctx->stream>>>(q, m, w, v, thI[0],
                                                                         thI[1]);
    MG_LAUNCH_CHECK(ctx);
    if constexpr (sizeof(T) == 4) {
      if ((pmode & 2) && g_mesh_bvh8 && s->depth8 >= 0)
        wf_shadow_p8_kernel<NCH><<<pgrid8, kMThreads, 0, ctx->stream>>>(m, w, v);
      else if ((pmode & 2) && sstk && g_mesh_qnodes)
        wf_shadow_p_kernel<NCH, true, true><<<pgrid, kMThreads, 0, ctx->stream>>>(m, w, v);
      else if ((pmode & 2) && sstk)
        wf_shadow_p_kernel<NCH, true><<<pgrid, kMThreads, 0, ctx->stream>>>(m, w, v);
      else if (pmode & 2)
        wf_shadow_p_kernel<NCH, false><<<pgrid, kMThreads, 0, ctx->stream>>>(m, w, v);
      else
        wf_shadow_kernel<T, NCH><<<grid, kMThreads, 0, ctx->stream>>>(m, w, v);
    } else {
      wf_shadow_kernel<T, NCH><<<grid, kMThreads, 0, ctx->stream>>>(m, w, v);
    }
    MG_LAUNCH_CHECK(ctx);
  }
  MG_NVTX("wavefront scatter");
  const int sgrid = grid_for(ctx, npix, kMThreads, 8);
  if (acc.ilv)
    wf_scatter_kernel<T, NCH, true><<<sgrid, kMThreads, 0, ctx->stream>>>(
        q, w, target_img, acc, ctx->partials, ctx->counter, loss_out, g_mesh_scatter_agg);
  else
    wf_scatter_kernel<T, NCH, false><<<sgrid, kMThreads, 0, ctx->stream>>>(
        q, w, target_img, acc, ctx->partials, ctx->counter, loss_out, g_mesh_scatter_agg);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

int dispatch_wavefront(mg_ctx* ctx, mg_mesh_scene* s, const MeshK& q, int32_t dtype, int nprop,
                       const void* target_img, const void* now, const void* prev,
                       const AccTable& tbl, double* loss_out) {
  if (dtype == MG_F64 && s->nch == 5)
    return wavefront_pair<double, 5>(ctx, s, q, nprop, (const double*)target_img,
                                     (const double*)now, (const double*)prev, tbl, loss_out);
  if (dtype == MG_F64)
    return wavefront_pair<double, 4>(ctx, s, q, nprop, (const double*)target_img,
                                     (const double*)now, (const double*)prev, tbl, loss_out);
  if (dtype == MG_F32 && s->nch == 5)
    return wavefront_pair<float, 5>(ctx, s, q, nprop, (const float*)target_img,
                                    (const float*)now, (const float*)prev, tbl, loss_out);
  if (dtype == MG_F32)
    return wavefront_pair<float, 4>(ctx, s, q, nprop, (const float*)target_img,
                                    (const float*)now, (const float*)prev, tbl, loss_out);
  return fail(MG_EINVAL, "mg_meshscene_sample_pair: unknown dtype");
}

}  // namespace mesh
}  // namespace mg

using namespace mg;
using namespace mg::mesh;

extern "C" {

int mg_meshscene_sample_pair(mg_ctx* ctx, mg_mesh_scene* s, int32_t dtype, int32_t W,
                             int32_t H, const double* view, const void* target_img,
                             const void* now, const void* prev, uint64_t key, uint32_t iteration,
                             int32_t row0, int32_t row1, int32_t prop_paths, void* accum,
                             void* prop, void* diff, double* loss_out) {
  MG_NVTX("mg_meshscene_sample_pair");
  if (!ctx || !s || !target_img || !now || !prev || !accum || !loss_out || (!prop != !diff))
    return fail(MG_EINVAL, "mg_meshscene_sample_pair: null argument");
  const bool keep_acc = !prop;  // pair left in accum for mg_meta_update_fixed
  if (prop_paths < 2 || prop_paths > kMaxProp)
    return fail(MG_EINVAL, "mg_meshscene_sample_pair: prop_paths must lie in [2, 8]");
  if (W < 1 || H < 1) return fail(MG_EINVAL, "mg_meshscene_sample_pair: bad sizes");
  if (row0 < 0 || row1 > H || row0 > row1)
    return fail(MG_EINVAL, "mg_meshscene_sample_pair: bad rows");
  int st = check_view(view);
  if (st) return st;
  MeshK q = make_k(s, W, H, view, key, iteration);
  q.it_offset = ctx->it_offset;
  q.row0 = row0;
  q.row1 = row1;
  const long long np = (long long)s->nobj * s->nch * s->R * s->R;
  unsigned long long* acc = (unsigned long long*)accum;
  AccTable tbl{};
  tbl.ptr[0] = acc;
  tbl.shard = int(np);
  tbl.ilv = 1;
  tbl.touch = keep_acc ? s->touch : nullptr;
  // the megakernel implements the configs[3] form (4 channels, 2 proportional
  // paths) and accumulates in planar order
  const bool mega = g_mesh_megakernel && s->nch == 4 && prop_paths == 2 && !keep_acc;
  if (mega) {
    s->last_now_slot = -1;  // the texel-copy reuse chain follows wavefront calls only
    st = megakernel_pair(ctx, s, q, dtype, target_img, now, prev, acc, np, loss_out);
  } else {
    st = dispatch_wavefront(ctx, s, q, dtype, prop_paths, target_img, now, prev, tbl, loss_out);
  }
  if (st) return st;
  if (keep_acc) return MG_OK;
  if (!mega) {
    const long long cells = (long long)s->nobj * s->R * s->R;
    if (dtype == MG_F64)
      return finalize_ilv<double>(ctx, s->nch, cells, s->R * s->R, acc, (double*)prop,
                                  (double*)diff);
    return finalize_ilv<float>(ctx, s->nch, cells, s->R * s->R, acc, (float*)prop, (float*)diff);
  }
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

// Tile-sharded form (fused scatter + reduce-scatter over peer memory): the
// partial pair of image rows [row0, row1) is accumulated straight into the
// owners' accumulators, acc_ptrs[r] = rank r's device int64 [2][shard]
// (prop | diff; peer pointers, e.g. torch symmetric memory).  No full-length
// partial buffers, no reduce-scatter launch: after a barrier each rank runs
// mg_fixed_finalize on its own shard.
int mg_meshscene_sample_pair_sharded(mg_ctx* ctx, mg_mesh_scene* s, int32_t dtype, int32_t W,
                                     int32_t H, const double* view, const void* target_img,
                                     const void* now, const void* prev, uint64_t key,
                                     uint32_t iteration, int32_t row0, int32_t row1,
                                     int32_t prop_paths, int32_t world, void* const* acc_ptrs,
                                     int64_t shard, double* loss_out) {
  if (!ctx || !s || !target_img || !now || !prev || !acc_ptrs || !loss_out)
    return fail(MG_EINVAL, "mg_meshscene_sample_pair_sharded: null argument");
  if (prop_paths < 2 || prop_paths > kMaxProp)
    return fail(MG_EINVAL, "mg_meshscene_sample_pair_sharded: prop_paths must lie in [2, 8]");
  if (W < 1 || H < 1 || row0 < 0 || row1 > H || row0 > row1)
    return fail(MG_EINVAL, "mg_meshscene_sample_pair_sharded: bad sizes or rows");
  const long long np = (long long)s->nobj * s->nch * s->R * s->R;
  if (world < 1 || world > kMaxRanks || shard < 1 || shard * world != np)
    return fail(MG_EINVAL, "mg_meshscene_sample_pair_sharded: world * shard must equal the "
                           "parameter count (1 <= world <= 8)");
  int st = check_view(view);
  if (st) return st;
  MeshK q = make_k(s, W, H, view, key, iteration);
  q.it_offset = ctx->it_offset;
  q.row0 = row0;
  q.row1 = row1;
  AccTable tbl{};
  for (int r = 0; r < world; ++r) {
    if (!acc_ptrs[r]) return fail(MG_EINVAL, "mg_meshscene_sample_pair_sharded: null accumulator");
    tbl.ptr[r] = static_cast<unsigned long long*>(acc_ptrs[r]);
  }
  tbl.shard = int(shard);
  tbl.ilv = 0;
  return dispatch_wavefront(ctx, s, q, dtype, prop_paths, target_img, now, prev, tbl, loss_out);
}

// Queue counters of the scene's last wavefront sample pair (diagnostics):
// out[0..kMaxV] = paths entering isect at each depth (entry kMaxV: bounce
// survivors of the last depth), out[kMaxV+1 .. 2kMaxV+1] = shadow rays per
// depth.  n_out >= 2 * (kMaxV + 1); synchronises the context's stream.
int mg_meshscene_queue_counts(mg_ctx* ctx, const mg_mesh_scene* s, int32_t n_out, uint32_t* out) {
  if (!ctx || !s || !out || n_out < 2 * (kMaxV + 1))
    return fail(MG_EINVAL, "mg_meshscene_queue_counts: bad arguments");
  if (!s->last_cnt) return fail(MG_EINVAL, "mg_meshscene_queue_counts: no wavefront call yet");
  MG_CUDA_TRY(cudaMemcpyAsync(out, s->last_cnt, sizeof(uint32_t) * 2 * (kMaxV + 1),
                              cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return MG_OK;
}

#ifndef MG_PREV_REUSE
#define MG_PREV_REUSE 1  // 0: ignore the opt-in (A/B builds)
#endif
int mg_meshscene_set_touch_map(mg_mesh_scene* s, uint32_t* touch_map) {
  if (!s) return fail(MG_EINVAL, "mg_meshscene_set_touch_map: null scene");
  s->touch = touch_map;
  return MG_OK;
}

int mg_meshscene_set_prev_reuse(mg_mesh_scene* s, int32_t enable) {
  if (!s) return fail(MG_EINVAL, "mg_meshscene_set_prev_reuse: null scene");
  s->prev_reuse = MG_PREV_REUSE && enable != 0;
  s->last_now_slot = -1;
  return MG_OK;
}

// Converts one rank's fixed-point accumulator [2][n] into prop / diff (dtype)
// and zeroes it.
int mg_fixed_finalize(mg_ctx* ctx, int32_t dtype, int64_t n, void* accum, void* prop,
                      void* diff) {
  if (!ctx || (n > 0 && (!accum || !prop || !diff)))
    return fail(MG_EINVAL, "mg_fixed_finalize: null argument");
  if (n <= 0) return MG_OK;
  const int fgrid = grid_for(ctx, n, 256, 8);
  unsigned long long* acc = static_cast<unsigned long long*>(accum);
  if (dtype == MG_F64)
    mesh_finalize_kernel<double><<<fgrid, 256, 0, ctx->stream>>>(n, acc, (double*)prop,
                                                                 (double*)diff);
  else if (dtype == MG_F32)
    mesh_finalize_kernel<float><<<fgrid, 256, 0, ctx->stream>>>(n, acc, (float*)prop,
                                                                (float*)diff);
  else
    return fail(MG_EINVAL, "mg_fixed_finalize: unknown dtype");
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

}  // extern "C"
