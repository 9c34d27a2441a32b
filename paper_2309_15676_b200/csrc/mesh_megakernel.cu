// Mesh renderer, one thread per pixel (the first design; kept as the A/B
// reference of the wavefront and for renders): paths A (both parameter
// sets), B and C traced in turn, path A's / B's per-vertex adjoint data in
// local memory, suffix radiance accumulated backwards, 2^-40 fixed-point
// atomics.  Warps take 32 pixels at a time from a global counter; the
// traversal, path and scatter bodies are out of line so the kernel's
// instruction footprint stays inside the I-cache.  Also: the render kernel
// (targets) and the closest-hit ray query.  DESIGN.md §12.
#include "mesh.cuh"

namespace mg {
namespace mesh {
namespace {

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
__device__ __noinline__ int mesh_path(const MeshK& q, const MeshDev& m, const float4* sn,
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
    const int slot = trace_t<false, T>(m, sn, o, d, INFINITY, t, bu, bv);
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
      if (trace_t<true, T>(m, sn, xo, w, wl - kOff, ts, tu, tv) < 0) {
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

template <class T, int NS>
__device__ __noinline__ void scatter(const PathStore<T, NS>& st, int nv, const T E[3], int s, const T w[3],
                        int R2, unsigned long long* __restrict__ acc) {
  T Q[3] = {E[0], E[1], E[2]};
  for (int v = nv - 1; v >= 0; --v) {
    T gr = T(0);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const T gb = w[c] * ((st.A[s][v][c] / T(kPiM)) + Q[c] * (st.invfb[s][v][c] / T(kPiM)));
      red_add_u64(&acc[st.base[v] + c * R2], fixq(double(gb)));
      gr += w[c] * (st.A[s][v][c] * st.dSn[s][v] + Q[c] * (st.invfb[s][v][c] * st.dSb[s][v]));
    }
    red_add_u64(&acc[st.base[v] + 3 * R2], fixq(double(gr)));
#pragma unroll
    for (int c = 0; c < 3; ++c) Q[c] = Q[c] + st.C[s][v][c];
  }
}

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
      mesh_path<T, 1, false, NoStore, NCH>(q, m, sn, th, px, py, 0xffffffffu, uint32_t(s),
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
  if (q.it_offset) q.iteration += __ldg(q.it_offset);
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
    mesh_path<T, 1, false, NoStore>(q, m, sn, th, px, py, q.iteration, 1u, LB, EB, nullptr);
    mesh_path<T, 2, false, NoStore>(q, m, sn, th, px, py, q.iteration, 2u, LC, EC, nullptr);
    T rA[3], rB[3], wC0[3], wC1[3];
    {
      PathStore<T, 2> st;
      const int na =
          mesh_path<T, 2, true>(q, m, sn, th, px, py, q.iteration, 0u, LA, EA, &st);
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
          mesh_path<T, 1, true>(q, m, sn, th, px, py, q.iteration, 1u, LB, EB, &st);
      scatter<T, 1>(st, nb, EB[0], 0, rA, R2, acc);
    }
  }
  Acc a;
  a.ssn = loss;
  grid_reduce4<kMThreads>(a.partials(), partials, counter,
                          [&](const ReducePartials& t) { *loss_out = t.ssn; });
}

__global__ void mesh_intersect_kernel(MeshDev m, int n, const double* __restrict__ rays,
                                      double* __restrict__ t_out, int* __restrict__ tri_out) {
  MESH_SMEM;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double o[3] = {rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]};
    const double d[3] = {rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5]};
    double t = INFINITY, u, v;
    const int s = trace<false>(m, sn, o, d, INFINITY, t, u, v);
    t_out[i] = s < 0 ? INFINITY : t;
    tri_out[i] = s < 0 ? -1 : m.orig[s];
  }
}

}  // namespace

int megakernel_pair(mg_ctx* ctx, mg_mesh_scene* s, const MeshK& q, int32_t dtype,
                    const void* target_img, const void* now, const void* prev,
                    unsigned long long* acc, long long np, double* loss_out) {
  const int grid = grid_for(ctx, int64_t(q.W) * (q.row1 - q.row0) + 1, kMThreads, 4);
  MG_CUDA_TRY(cudaMemsetAsync(s->work, 0, sizeof(unsigned int), ctx->stream));
  if (dtype == MG_F64)
    mesh_pair_kernel<double><<<grid, kMThreads, 0, ctx->stream>>>(
        q, dev_of(s), (const double*)target_img, (const double*)now, (const double*)prev, acc, np,
        s->work, ctx->partials, ctx->counter, loss_out);
  else if (dtype == MG_F32)
    mesh_pair_kernel<float><<<grid, kMThreads, 0, ctx->stream>>>(
        q, dev_of(s), (const float*)target_img, (const float*)now, (const float*)prev, acc, np,
        s->work, ctx->partials, ctx->counter, loss_out);
  else
    return fail(MG_EINVAL, "mg_meshscene_sample_pair: unknown dtype");
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

}  // namespace mesh
}  // namespace mg

using namespace mg;
using namespace mg::mesh;

extern "C" {

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

}  // extern "C"
