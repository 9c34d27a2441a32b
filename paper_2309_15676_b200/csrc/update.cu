// Fused estimator/optimiser kernels.
//
// mg_meta_update is THE hot kernel: one HBM pass that fuses
//   Moment2(beta_f).step(prop)                 moment2.hpp:30-39 (harness.cpp:144)
//   decoupled diff variance + Moment2(beta_d)  harness.cpp:145-158, meta.hpp:51-53
//   MetaEstimator::step                        meta.hpp:90-113 (harness.cpp:160)
//   params += delta; project                   harness.cpp:182-188, problems.cpp:228
//   sum (dp)^2, #changed, sum (p-T)^2, #nonfinite  problems.cpp:206,214,225; harness.cpp:116
// The reference evaluates these as ~12 Eigen statements (~12 memory passes
// plus temporaries); here every parameter is touched once: 8 streams read,
// 6 written (56 B/param fp32, 112 B/param fp64), the reductions ride along in
// registers and finish in the last CTA (deterministic fixed-order tree).
//
// Arithmetic follows the reference expression by expression (same operand
// order, no FMA: the library is built with --fmad=false), so the fp64 path is
// bit-identical to the oracle for the elementwise outputs.
#include <math.h>

#include <string>
#include <type_traits>

#include "mg_common.cuh"
#include "tma.cuh"
#include "meta_math.cuh"

namespace mg {
// Test/benchmark switch: force the register-streaming kernel (mg_set_option).
bool g_disable_tma = false;
extern bool g_render_vec;
extern bool g_render_fast;
extern bool g_cluster_runner;
extern uint64_t g_pool_keep;
int apply_pool_keep(int device);
extern int g_render_fast_variant;
int render_fast_variants();
extern bool g_mesh_megakernel;
extern int g_mesh_persistent;
extern int g_mesh_tail;
extern bool g_mesh_scatter_agg;
extern bool g_mesh_bvh8;
extern bool g_mesh_smem_stack;
extern bool g_mesh_qnodes;
extern bool g_helix_split;
extern int g_bvh_leaf;
extern int g_bvh_axes;
extern int g_bvh_bins;
// -1: per-dtype default measured on B200: fp32 -> variant 8 (1 CTA/SM x 640
// threads, 2 stages of 10 KB tiles: 20 warps to issue the body and ~180 KB
// in flight; interleaved A/B over 30 blocks of 20 launches,
// tools/ab_update_variants.py: 2.31 ms at 2^28 against 2.52 for round 1's
// variant 6, whose pick came from a sequential sweep that the launch-to-
// launch drift of HBM biased), fp64 -> variant 9 (1 CTA/SM x 512 threads,
// 2 stages of 8 KB tiles: 4.63 ms against 5.4-5.7 for variant 0).
int g_tma_variant = -1;
namespace {

constexpr int kThreads = 256;

template <class T, bool FIRST, bool VEC>
__global__ void __launch_bounds__(kThreads)
    meta_update_kernel(int64_t n, MetaK k, MetaPtrs<T> q, mg_update_scalars* sc,
                       ReducePartials* partials, unsigned int* counter) {
  const StepScal s = load_step_scalars(k, sc);
  const bool has_target = q.target != nullptr;
  Acc acc;
  const int64_t tid = int64_t(blockIdx.x) * kThreads + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * kThreads;
  constexpr int W = VEC ? VecOf<T>::width : 1;
  const int64_t items = VEC ? n / W : 0;
  if constexpr (VEC) {
    const bool pp = k.diff_norm == MG_DIFF_NORM_PER_PARAM;
    for (int64_t it = tid; it < items; it += stride) {
      const int64_t b = it * W;
      const Pack<T> P = ld_stream(q.prop + b);
      const Pack<T> D = ld_stream(q.diff + b);
      const Pack<T> VP = q.vprop ? ld_stream(q.vprop + b) : P;
      const Pack<T> VD = q.vdiff ? ld_stream(q.vdiff + b) : D;
      Pack<T> M2P{}, M2D{}, ME{}, VA{}, AP{}, PO, DL;
      if (!FIRST) {
        M2P = ld_plain(q.m2p + b);
        ME = ld_plain(q.mean + b);
        VA = ld_plain(q.var + b);
        AP = ld_plain(q.ap + b);
      }
      if (s.cnt0 > 0) M2D = ld_plain(q.m2d + b);
      const Pack<T> PI = ld_plain(q.pin + b);
      Pack<T> PP{}, TG{};
      if (pp) PP = ld_plain(q.pprev + b);
      if (has_target) TG = ld_plain(q.target + b);
#pragma unroll
      for (int w = 0; w < W; ++w)
        meta_elem<T, FIRST>(k, s, P.v[w], D.v[w], VP.v[w], VD.v[w], M2P.v[w], M2D.v[w], ME.v[w],
                            VA.v[w], AP.v[w], PI.v[w], PP.v[w], TG.v[w], has_target, PO.v[w],
                            DL.v[w], acc);
      st_stream(q.m2p + b, M2P);
      if (s.active) st_stream(q.m2d + b, M2D);
      st_stream(q.mean + b, ME);
      st_stream(q.var + b, VA);
      st_stream(q.ap + b, AP);
      st_stream(q.pout + b, PO);
      if (q.delta) st_stream(q.delta + b, DL);
    }
  }
  // scalar path: everything (unaligned) or the tail (aligned)
  for (int64_t i = items * W + tid; i < n; i += stride) {
    const T P = q.prop[i], D = q.diff[i];
    const T VP = q.vprop ? q.vprop[i] : P;
    const T VD = q.vdiff ? q.vdiff[i] : D;
    T M2P = FIRST ? T(0) : q.m2p[i];
    T M2D = s.cnt0 > 0 ? q.m2d[i] : T(0);
    T ME = FIRST ? T(0) : q.mean[i];
    T VA = FIRST ? T(0) : q.var[i];
    T AP = FIRST ? T(0) : q.ap[i];
    const T PI = q.pin[i];
    const T PP = k.diff_norm == MG_DIFF_NORM_PER_PARAM ? q.pprev[i] : T(0);
    const T TG = has_target ? q.target[i] : T(0);
    T PO, DL;
    meta_elem<T, FIRST>(k, s, P, D, VP, VD, M2P, M2D, ME, VA, AP, PI, PP, TG, has_target, PO, DL,
                        acc);
    q.m2p[i] = M2P;
    if (s.active) q.m2d[i] = M2D;
    q.mean[i] = ME;
    q.var[i] = VA;
    q.ap[i] = AP;
    q.pout[i] = PO;
    if (q.delta) q.delta[i] = DL;
  }
  grid_reduce4<kThreads>(acc.partials(), partials, counter, [&](const ReducePartials& t) {
    sc->ssn = t.ssn;
    sc->changed = t.changed;
    sc->loss = has_target ? t.loss : nan("");
    sc->nonfinite = t.nonfinite;
    sc->diff_count = s.cnt;
    sc->diff_decay_pow = s.dpow;
    sc->prop_decay_pow = s.ppow;
    sc->ssn_used = s.ssn;
  });
}

// --------------------------------------------- TMA-pipelined fused update
// Persistent variant for the common case (global diff norm, no independent
// variance pair): every CTA streams 4 KB tiles of up to 9 input arrays into a
// kStages-deep shared-memory ring with 1-D bulk copies (cp.async.bulk +
// mbarrier complete_tx), so ~100 KB per SM are in flight regardless of
// register pressure; the 6 outputs are written straight from registers.
constexpr int kTmaArrays = 9;  // prop diff m2p m2d mean var ap pin target

// Schedules of the TMA pipeline (threads per CTA, ring depth, CTAs per SM);
// the tile is one 16-byte pack per thread per array.  Selected with
// mg_set_option("tma_variant", i); default g_tma_variant.
struct TmaVariant {
  int threads, stages, ctas_per_sm;
};
__host__ __device__ constexpr TmaVariant tma_variant(int i) {
  return i == 0 ? TmaVariant{256, 4, 1}
       : i == 1 ? TmaVariant{256, 3, 2}
       : i == 2 ? TmaVariant{512, 3, 1}
       : i == 3 ? TmaVariant{768, 2, 1}
       : i == 4 ? TmaVariant{256, 2, 3}
       : i == 5 ? TmaVariant{160, 5, 2}
       : i == 6 ? TmaVariant{192, 4, 2}
       : i == 7 ? TmaVariant{224, 3, 2}
       : i == 8 ? TmaVariant{640, 2, 1}
                : TmaVariant{512, 2, 1};
}
constexpr int kNumTmaVariants = 10;

template <class T, int THREADS>
__host__ __device__ constexpr int tma_tile() { return THREADS * VecOf<T>::width; }
template <class T, int THREADS, int STAGES>
constexpr size_t tma_smem_bytes() {
  return size_t(STAGES) * kTmaArrays * tma_tile<T, THREADS>() * sizeof(T);
}

template <class T, bool FIRST, int kTmaThreads, int kTmaStages, int kMinBlocks>
__global__ void __launch_bounds__(kTmaThreads, kMinBlocks)
    meta_update_tma_kernel(int64_t n, MetaK k, MetaPtrs<T> q, mg_update_scalars* sc,
                           ReducePartials* partials, unsigned int* counter) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kTmaStages];
  constexpr int TILE = tma_tile<T, kTmaThreads>();
  constexpr int W = VecOf<T>::width;
  static_assert(TILE == kTmaThreads * W, "one 16-byte pack per thread per array");
  T* sbuf = reinterpret_cast<T*>(smem_raw);
  const StepScal s = load_step_scalars(k, sc);
  const bool has_target = q.target != nullptr;
  const T* src[kTmaArrays] = {q.prop, q.diff, q.m2p, q.m2d, q.mean, q.var, q.ap, q.pin, q.target};
  const bool use[kTmaArrays] = {true,  true,  !FIRST, s.cnt0 > 0, !FIRST,
                                !FIRST, !FIRST, true,  has_target};
  uint32_t tx = 0;
#pragma unroll
  for (int a = 0; a < kTmaArrays; ++a) tx += use[a] ? uint32_t(TILE * sizeof(T)) : 0u;

  const int64_t tiles = n / TILE;
  const int64_t my_tiles =
      int64_t(blockIdx.x) < tiles ? (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kTmaStages; ++st) mbar_init(&full[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = l2_evict_first_policy();
  auto issue = [&](int64_t li) {  // thread 0 only
    const int st = int(li % kTmaStages);
    const int64_t tile = int64_t(blockIdx.x) + li * gridDim.x;
    MG_DCHECK((tile + 1) * TILE <= n && st < kTmaStages);
    mbar_arrive_expect_tx(&full[st], tx);
#pragma unroll
    for (int a = 0; a < kTmaArrays; ++a)
      if (use[a])
        bulk_g2s_hint(sbuf + (size_t(st) * kTmaArrays + a) * TILE, src[a] + tile * TILE,
                      uint32_t(TILE * sizeof(T)), &full[st], pol);
  };
  if (threadIdx.x == 0)
    for (int64_t li = 0; li < my_tiles && li < kTmaStages; ++li) issue(li);

  Acc acc;
  const int e = threadIdx.x * W;
  for (int64_t li = 0; li < my_tiles; ++li) {
    const int st = int(li % kTmaStages);
    mbar_wait(&full[st], uint32_t((li / kTmaStages) & 1));
    const T* sb = sbuf + size_t(st) * kTmaArrays * TILE + e;
    const Pack<T> P = ld_plain(sb + 0 * TILE);
    const Pack<T> D = ld_plain(sb + 1 * TILE);
    Pack<T> M2P{}, M2D{}, ME{}, VA{}, AP{}, TG{}, PO, DL;
    if (!FIRST) {
      M2P = ld_plain(sb + 2 * TILE);
      ME = ld_plain(sb + 4 * TILE);
      VA = ld_plain(sb + 5 * TILE);
      AP = ld_plain(sb + 6 * TILE);
    }
    if (s.cnt0 > 0) M2D = ld_plain(sb + 3 * TILE);
    const Pack<T> PI = ld_plain(sb + 7 * TILE);
    if (has_target) TG = ld_plain(sb + 8 * TILE);
#pragma unroll
    for (int w = 0; w < W; ++w) {
#if MG_TMA_NOMATH  // probe builds only: the same traffic without the arithmetic
      M2P.v[w] += P.v[w];
      M2D.v[w] += D.v[w];
      ME.v[w] += P.v[w];
      VA.v[w] += D.v[w];
      AP.v[w] += P.v[w];
      PO.v[w] = PI.v[w] + D.v[w];
#else
      meta_elem<T, FIRST>(k, s, P.v[w], D.v[w], P.v[w], D.v[w], M2P.v[w], M2D.v[w], ME.v[w],
                          VA.v[w], AP.v[w], PI.v[w], T(0), TG.v[w], has_target, PO.v[w], DL.v[w],
                          acc);
#endif
    }
    const int64_t b = (int64_t(blockIdx.x) + li * gridDim.x) * TILE + e;
    // streaming (evict-first) stores: the state is re-read only next step,
    // long after a 2^28-parameter pass has cycled L2 (A/B: 2.62 -> 2.54 ms)
    st_stream(q.m2p + b, M2P);
    if (s.active) st_stream(q.m2d + b, M2D);
    st_stream(q.mean + b, ME);
    st_stream(q.var + b, VA);
    st_stream(q.ap + b, AP);
    st_stream(q.pout + b, PO);
    if (q.delta) st_stream(q.delta + b, DL);
    __syncthreads();  // every thread is done reading stage st
    if (threadIdx.x == 0 && li + kTmaStages < my_tiles) {
      fence_proxy_async_smem();
      issue(li + kTmaStages);
    }
  }
  // tail elements [tiles*TILE, n)
  const int64_t tid = int64_t(blockIdx.x) * kTmaThreads + threadIdx.x;
  for (int64_t i = tiles * TILE + tid; i < n; i += int64_t(gridDim.x) * kTmaThreads) {
    const T P = q.prop[i], D = q.diff[i];
    T M2P = FIRST ? T(0) : q.m2p[i];
    T M2D = s.cnt0 > 0 ? q.m2d[i] : T(0);
    T ME = FIRST ? T(0) : q.mean[i];
    T VA = FIRST ? T(0) : q.var[i];
    T AP = FIRST ? T(0) : q.ap[i];
    const T PI = q.pin[i];
    const T TG = has_target ? q.target[i] : T(0);
    T PO, DL;
    meta_elem<T, FIRST>(k, s, P, D, P, D, M2P, M2D, ME, VA, AP, PI, T(0), TG, has_target, PO, DL,
                        acc);
    q.m2p[i] = M2P;
    if (s.active) q.m2d[i] = M2D;
    q.mean[i] = ME;
    q.var[i] = VA;
    q.ap[i] = AP;
    q.pout[i] = PO;
    if (q.delta) q.delta[i] = DL;
  }
  grid_reduce4<kTmaThreads>(acc.partials(), partials, counter, [&](const ReducePartials& t) {
    sc->ssn = t.ssn;
    sc->changed = t.changed;
    sc->loss = has_target ? t.loss : nan("");
    sc->nonfinite = t.nonfinite;
    sc->diff_count = s.cnt;
    sc->diff_decay_pow = s.dpow;
    sc->prop_decay_pow = s.ppow;
    sc->ssn_used = s.ssn;
  });
}

// ------------------------------ fused update from a fixed-point accumulator
// The mesh renderers' adjoints arrive as a texel-interleaved 2^-40
// fixed-point accumulator [cell = obj*R2 + texel][prop | diff][NCH] (int64);
// the parameters stay planar [obj][ch][texel].  This kernel converts,
// zeroes and consumes the accumulator in the same pass as the meta update,
// so the planar prop / diff arrays of mesh_finalize_ilv_kernel are never
// written nor read back: 16 B of HBM traffic less per parameter.  A tile is
// K = THREADS texels of one object: the accumulator tile (K x 2 x NCH words,
// contiguous) and, per state array, NCH contiguous K-runs (one per channel
// plane) arrive by 1-D bulk copies into a STAGES-deep ring (lanes of warp 0
// issue them in parallel); thread t owns texel t's NCH parameters, reads
// its fixed-point words from shared memory, zeroes the global tile with
// coalesced 16-byte stores and writes its outputs (coalesced per channel
// plane).  prop/diff = T(double(word) / 2^40), exactly mesh_finalize's
// conversion, so every element equals finalize + mg_meta_update's.
constexpr double kFixScale = 1099511627776.0;  // 2^40 (mesh.cuh kFixM)
constexpr int kFixArrays = 6;                   // m2p m2d mean var ap pin

template <class T, int NCH, int K>
__host__ __device__ constexpr size_t fix_stage_bytes() {
  return size_t(K) * 2 * NCH * 8 + size_t(kFixArrays) * NCH * K * sizeof(T);
}

// Thread t owns texels t, t + THREADS, ... (TPT of them): the tile is
// K = THREADS * TPT texels, so each channel run is one K-element copy.
// (16-byte packs of 4 consecutive texels per thread, i.e. 4x fewer threads
// for the same smem, measured 10-40 % slower: too few warps for the IEEE
// division chains.)
//
// TOUCH: a bit per texel cell says whether the cell's accumulator words may
// be non-zero (the mesh scatter sets it with every vertex it adds).  Most
// cells of a large texture set see no path in an iteration, so instead of
// one bulk copy of the whole accumulator tile, thread t fetches its own
// cell (NCH 16-byte cp.async's into the same stage, their completion
// counted on the stage's mbarrier) only if its bit is set — otherwise it
// writes zeros to the stage — and zeroes the global cell only if it read
// it; the tile's bits are cleared.  32 B/param of accumulator traffic
// become 32 B per TOUCHED parameter's sectors.
template <class T, bool FIRST, bool TOUCH, int NCH, int THREADS, int TPT, int STAGES, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
    meta_update_fixed_tma_kernel(int64_t tiles, int R2, MetaK k, MetaPtrs<T> q,
                                 unsigned long long* __restrict__ acc,
                                 unsigned int* __restrict__ touch, mg_update_scalars* sc,
                                 ReducePartials* partials, unsigned int* counter) {
  static_assert(!TOUCH || (TPT == 1 && THREADS % 32 == 0), "touch map: one cell per thread");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES];
  constexpr int K = THREADS * TPT;
  constexpr size_t kAccBytes = size_t(K) * 2 * NCH * 8;
  constexpr size_t kStage = fix_stage_bytes<T, NCH, K>();
  const StepScal s = load_step_scalars(k, sc);
  T* const dst_arr[kFixArrays] = {q.m2p, q.m2d, q.mean, q.var, q.ap, nullptr};
  const T* const src_arr[kFixArrays] = {q.m2p, q.m2d, q.mean, q.var, q.ap, q.pin};
  const bool use[kFixArrays] = {!FIRST, s.cnt0 > 0, !FIRST, !FIRST, !FIRST, true};
  (void)dst_arr;
  uint32_t tx = TOUCH ? 0u : uint32_t(kAccBytes);
  int ncopy = 1;
#pragma unroll
  for (int a = 0; a < kFixArrays; ++a)
    if (use[a]) {
      tx += uint32_t(NCH * K * sizeof(T));
      ncopy += NCH;
    }
  const int64_t my_tiles =
      int64_t(blockIdx.x) < tiles ? (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < STAGES; ++st) mbar_init(&full[st], TOUCH ? 1 + THREADS : 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = l2_evict_first_policy();
  constexpr int kCellVecs = 2 * NCH * 8 / 16;  // 16-byte pieces of one cell
  // TOUCH: the bits of local tile li (one word per warp)
  auto tile_bits = [&](int64_t li) -> unsigned {
    const int64_t cell0 = (int64_t(blockIdx.x) + li * gridDim.x) * K;
    return touch[(cell0 + threadIdx.x) >> 5];
  };
  // TOUCH: every thread brings its own cell of local tile li into the stage
  auto issue_cell = [&](int64_t li, unsigned bits) {
    const int st = int(li % STAGES);
    const int64_t cell0 = (int64_t(blockIdx.x) + li * gridDim.x) * K;
    uint4* dst = reinterpret_cast<uint4*>(smem_raw + size_t(st) * kStage) +
                 size_t(threadIdx.x) * kCellVecs;
    if ((bits >> (threadIdx.x & 31)) & 1u) {
      const uint4* src = reinterpret_cast<const uint4*>(acc + (cell0 + threadIdx.x) * 2 * NCH);
#pragma unroll
      for (int u = 0; u < kCellVecs; ++u) cp_async_16(dst + u, src + u);
      cp_async_mbar_arrive_noinc(&full[st]);
    } else {
#pragma unroll
      for (int u = 0; u < kCellVecs; ++u) dst[u] = make_uint4(0u, 0u, 0u, 0u);
      mbar_arrive(&full[st]);
    }
  };
  // warp 0: lane 0 arms the stage's barrier, lanes 0..ncopy-1 issue one copy each
  auto issue = [&](int64_t li) {
    const int st = int(li % STAGES);
    const int64_t tile = int64_t(blockIdx.x) + li * gridDim.x;
    const int64_t cell0 = tile * K;
    const int64_t obj = cell0 / R2, tex0 = cell0 - obj * R2;
    unsigned char* sb = smem_raw + size_t(st) * kStage;
    const int lane = int(threadIdx.x);
    if (lane == 0) mbar_arrive_expect_tx(&full[st], tx);
    __syncwarp();
    if (lane == 0) {
      if (!TOUCH) bulk_g2s_hint(sb, acc + cell0 * 2 * NCH, uint32_t(kAccBytes), &full[st], pol);
    } else if (lane < ncopy) {
      // lane j >= 1: the (j-1)-th used (array, channel) run
      int r = lane - 1, a = 0;
#pragma unroll
      for (int b = 0; b < kFixArrays; ++b)
        if (use[b]) {
          if (r >= NCH) {
            r -= NCH;
          } else {
            a = b;
            break;
          }
        }
      const int c = r;
      T* dst = reinterpret_cast<T*>(sb + kAccBytes) + (size_t(a) * NCH + c) * K;
      bulk_g2s_hint(dst, src_arr[a] + (obj * NCH + c) * int64_t(R2) + tex0,
                    uint32_t(K * sizeof(T)), &full[st], pol);
    }
  };
  // the bits of the tiles in flight (their cells are zeroed / their words
  // cleared when the tile is consumed) and of the next tile to issue
  unsigned bits_ring[STAGES];
#pragma unroll
  for (int st = 0; st < STAGES; ++st) bits_ring[st] = 0u;
  for (int64_t li = 0; li < my_tiles && li < STAGES; ++li) {
    if (threadIdx.x < 32) issue(li);
    if constexpr (TOUCH) {
      const unsigned b = tile_bits(li);
#pragma unroll
      for (int st = 0; st < STAGES; ++st)
        if (st == int(li)) bits_ring[st] = b;
      issue_cell(li, b);
    }
  }

  Acc red;
  const int t = int(threadIdx.x);
  for (int64_t li = 0; li < my_tiles; ++li) {
    const int st = int(li % STAGES);
    unsigned bits_now = 0u, bits_next = 0u;
    if constexpr (TOUCH) {
#pragma unroll
      for (int s2 = 0; s2 < STAGES; ++s2)
        if (s2 == st) bits_now = bits_ring[s2];
      // requested now, used after this tile's arithmetic
      if (li + STAGES < my_tiles) bits_next = tile_bits(li + STAGES);
    }
    mbar_wait(&full[st], uint32_t((li / STAGES) & 1));
    const unsigned char* sb = smem_raw + size_t(st) * kStage;
    const int64_t tile = int64_t(blockIdx.x) + li * gridDim.x;
    const int64_t cell0 = tile * K;
    const int64_t obj = cell0 / R2, tex0 = cell0 - obj * R2;
    // zero the global accumulator tile (its words are in shared memory now)
    if constexpr (TOUCH) {
      if ((bits_now >> (t & 31)) & 1u) {
        uint4* g = reinterpret_cast<uint4*>(acc + (cell0 + t) * 2 * NCH);
#pragma unroll
        for (int u = 0; u < kCellVecs; ++u) g[u] = make_uint4(0u, 0u, 0u, 0u);
      }
      if ((t & 31) == 0 && bits_now) touch[(cell0 + t) >> 5] = 0u;
    } else {
      uint4* g = reinterpret_cast<uint4*>(acc + cell0 * 2 * NCH);
#pragma unroll
      for (int u = 0; u < NCH * TPT; ++u) g[t + u * THREADS] = make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int j = 0; j < TPT; ++j) {
      const int tt = t + j * THREADS;
      const long long* aw = reinterpret_cast<const long long*>(sb) + size_t(tt) * 2 * NCH;
      const T* sv = reinterpret_cast<const T*>(sb + kAccBytes) + tt;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const T P = T(double(aw[c]) / kFixScale);
        const T D = T(double(aw[NCH + c]) / kFixScale);
        T M2P = FIRST ? T(0) : sv[(0 * NCH + c) * K];
        T M2D = s.cnt0 > 0 ? sv[(1 * NCH + c) * K] : T(0);
        T ME = FIRST ? T(0) : sv[(2 * NCH + c) * K];
        T VA = FIRST ? T(0) : sv[(3 * NCH + c) * K];
        T AP = FIRST ? T(0) : sv[(4 * NCH + c) * K];
        const T PI = sv[(5 * NCH + c) * K];
        T PO, DL;
        meta_elem<T, FIRST>(k, s, P, D, P, D, M2P, M2D, ME, VA, AP, PI, T(0), T(0), false, PO,
                            DL, red);
        const int64_t i = (obj * NCH + c) * int64_t(R2) + tex0 + tt;
        __stcs(q.m2p + i, M2P);
        if (s.active) __stcs(q.m2d + i, M2D);
        __stcs(q.mean + i, ME);
        __stcs(q.var + i, VA);
        __stcs(q.ap + i, AP);
        __stcs(q.pout + i, PO);
      }
    }
    __syncthreads();  // every thread is done reading stage st
    if (li + STAGES < my_tiles) {
      if (threadIdx.x < 32) {
        fence_proxy_async_smem();
        issue(li + STAGES);
      }
      if constexpr (TOUCH) {
#pragma unroll
        for (int s2 = 0; s2 < STAGES; ++s2)
          if (s2 == st) bits_ring[s2] = bits_next;
        issue_cell(li + STAGES, bits_next);
      }
    }
  }
  grid_reduce4<THREADS>(red.partials(), partials, counter, [&](const ReducePartials& r) {
    sc->ssn = r.ssn;
    sc->changed = r.changed;
    sc->loss = nan("");
    sc->nonfinite = r.nonfinite;
    sc->diff_count = s.cnt;
    sc->diff_decay_pow = s.dpow;
    sc->prop_decay_pow = s.ppow;
    sc->ssn_used = s.ssn;
  });
}

// Any shape / alignment / extras: one thread per parameter, the two
// fixed-point words read (and zeroed) straight from the accumulator.
template <class T, bool FIRST>
__global__ void __launch_bounds__(kThreads)
    meta_update_fixed_kernel(int64_t n, int nch, int R2, MetaK k, MetaPtrs<T> q,
                             unsigned long long* __restrict__ acc, mg_update_scalars* sc,
                             ReducePartials* partials, unsigned int* counter) {
  const StepScal s = load_step_scalars(k, sc);
  const bool has_target = q.target != nullptr;
  Acc red;
  for (int64_t i = int64_t(blockIdx.x) * kThreads + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * kThreads) {
    const int64_t plane = i / R2, tex = i - plane * R2;
    const int64_t obj = plane / nch, c = plane - obj * nch;
    unsigned long long* w = acc + (obj * R2 + tex) * 2 * nch + c;
    const T P = T(double((long long)w[0]) / kFixScale);
    const T D = T(double((long long)w[nch]) / kFixScale);
    w[0] = 0ull;
    w[nch] = 0ull;
    T M2P = FIRST ? T(0) : q.m2p[i];
    T M2D = s.cnt0 > 0 ? q.m2d[i] : T(0);
    T ME = FIRST ? T(0) : q.mean[i];
    T VA = FIRST ? T(0) : q.var[i];
    T AP = FIRST ? T(0) : q.ap[i];
    const T PI = q.pin[i];
    const T PP = k.diff_norm == MG_DIFF_NORM_PER_PARAM ? q.pprev[i] : T(0);
    const T TG = has_target ? q.target[i] : T(0);
    T PO, DL;
    meta_elem<T, FIRST>(k, s, P, D, P, D, M2P, M2D, ME, VA, AP, PI, PP, TG, has_target, PO, DL,
                        red);
    q.m2p[i] = M2P;
    if (s.active) q.m2d[i] = M2D;
    q.mean[i] = ME;
    q.var[i] = VA;
    q.ap[i] = AP;
    q.pout[i] = PO;
    if (q.delta) q.delta[i] = DL;
  }
  grid_reduce4<kThreads>(red.partials(), partials, counter, [&](const ReducePartials& r) {
    sc->ssn = r.ssn;
    sc->changed = r.changed;
    sc->loss = has_target ? r.loss : nan("");
    sc->nonfinite = r.nonfinite;
    sc->diff_count = s.cnt;
    sc->diff_decay_pow = s.dpow;
    sc->prop_decay_pow = s.ppow;
    sc->ssn_used = s.ssn;
  });
}

// ------------------------------------- shared-parameter fused step (peers)
// One rank's part of a tile-sharded shared-parameter iteration (SURVEY.md
// §8(e), configs 4/5 shape) as ONE kernel over NVLink peer memory: for its
// parameter shard it sums the ranks' partial sample pairs straight out of
// their buffers (reduce-scatter, rank order 0..G-1: deterministic), runs the
// fused meta update, and stores the new parameters into every rank's
// parameter buffer (all-gather by peer stores).  No staging copies; the only
// other collective is the 4-double scalar all-reduce.
constexpr int kMaxPeers = 8;
template <class T>
struct PeerPtrs {
  const T* prop[kMaxPeers];
  const T* diff[kMaxPeers];
  T* params_out[kMaxPeers];
};

template <class T, bool FIRST>
__global__ void __launch_bounds__(kThreads)
    shared_meta_update_kernel(int64_t n, int64_t lo, int world, MetaK k, PeerPtrs<T> pp,
                              const T* __restrict__ pin, T* __restrict__ m2p,
                              T* __restrict__ m2d, T* __restrict__ mean, T* __restrict__ var,
                              T* __restrict__ ap, const T* __restrict__ target,
                              mg_update_scalars* sc, ReducePartials* partials,
                              unsigned int* counter) {
  const StepScal s = load_step_scalars(k, sc);
  const bool has_target = target != nullptr;
  Acc acc;
  for (int64_t i = int64_t(blockIdx.x) * kThreads + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * kThreads) {
    const int64_t g = lo + i;
    T prop = pp.prop[0][g], diff = pp.diff[0][g];
    for (int q = 1; q < world; ++q) {  // reduce-scatter from the peers, fixed order
      prop = prop + pp.prop[q][g];
      diff = diff + pp.diff[q][g];
    }
    T M2P = FIRST ? T(0) : m2p[i];
    T M2D = s.cnt0 > 0 ? m2d[i] : T(0);
    T ME = FIRST ? T(0) : mean[i];
    T VA = FIRST ? T(0) : var[i];
    T AP = FIRST ? T(0) : ap[i];
    T PO, DL;
    meta_elem<T, FIRST>(k, s, prop, diff, prop, diff, M2P, M2D, ME, VA, AP, pin[g], T(0),
                        has_target ? target[i] : T(0), has_target, PO, DL, acc);
    m2p[i] = M2P;
    if (s.active) m2d[i] = M2D;
    mean[i] = ME;
    var[i] = VA;
    ap[i] = AP;
    for (int q = 0; q < world; ++q) pp.params_out[q][g] = PO;  // all-gather by peer stores
  }
  grid_reduce4<kThreads>(acc.partials(), partials, counter, [&](const ReducePartials& t) {
    sc->ssn = t.ssn;
    sc->changed = t.changed;
    sc->loss = has_target ? t.loss : nan("");
    sc->nonfinite = t.nonfinite;
    sc->diff_count = s.cnt;
    sc->diff_decay_pow = s.dpow;
    sc->prop_decay_pow = s.ppow;
    sc->ssn_used = s.ssn;
  });
}

// ------------------------------------------------------------------- Adam
struct AdamK {
  double beta1, beta2, c1, c2, d1, d2, lr, eps, proj_lo;
  int project;
};

template <class T>
__device__ __forceinline__ void adam_elem(const AdamK& k, T g, T& m, T& v, T pin, T target,
                                          bool has_target, T& pout, T& delta,
                                          Acc& acc) {
  m = T(k.beta1) * m + T(k.c1) * g;          // adam.hpp:32
  v = T(k.beta2) * v + T(k.c2) * (g * g);    // adam.hpp:33
  const T mh = div_z(m, T(k.d1));            // adam.hpp:34
  const T vh = div_z(v, T(k.d2));            // adam.hpp:35
  delta = div_z(T(-k.lr) * mh, sqrt_z(vh) + T(k.eps));  // adam.hpp:36  (div_z/sqrt_z: meta_math.cuh)
  T p = pin + delta;
  if (k.project) p = std_max(p, T(k.proj_lo));
  pout = p;
  const double d = double(p - pin);
  acc.ssn += d * d;
  acc.changed += (p != pin) ? 1u : 0u;
  if (has_target) {
    const double e = double(p - target);
    acc.loss += e * e;
  }
  acc.nonfinite += isfinite(p) ? 0u : 1u;
}

template <class T, bool FIRST, bool VEC>
__global__ void __launch_bounds__(kThreads)
    adam_update_kernel(int64_t n, AdamK k, const T* __restrict__ grad, T* __restrict__ m,
                       T* __restrict__ v, const T* pin, T* pout, const T* __restrict__ target,
                       T* __restrict__ delta, mg_update_scalars* sc, ReducePartials* partials,
                       unsigned int* counter) {
  const double ssn_in = __ldcg(&sc->ssn);
  const bool has_target = target != nullptr;
  Acc acc;
  const int64_t tid = int64_t(blockIdx.x) * kThreads + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * kThreads;
  constexpr int W = VEC ? VecOf<T>::width : 1;
  const int64_t items = VEC ? n / W : 0;
  if constexpr (VEC) {
    for (int64_t it = tid; it < items; it += stride) {
      const int64_t b = it * W;
      const Pack<T> G = ld_stream(grad + b);
      Pack<T> M{}, V{}, PO, DL, TG{};
      if (!FIRST) {
        M = ld_plain(m + b);
        V = ld_plain(v + b);
      }
      const Pack<T> PI = ld_plain(pin + b);
      if (has_target) TG = ld_plain(target + b);
#pragma unroll
      for (int w = 0; w < W; ++w)
        adam_elem<T>(k, G.v[w], M.v[w], V.v[w], PI.v[w], TG.v[w], has_target, PO.v[w], DL.v[w],
                     acc);
      st_stream(m + b, M);
      st_stream(v + b, V);
      st_stream(pout + b, PO);
      if (delta) st_stream(delta + b, DL);
    }
  }
  for (int64_t i = items * W + tid; i < n; i += stride) {
    T M = FIRST ? T(0) : m[i], V = FIRST ? T(0) : v[i], PO, DL;
    adam_elem<T>(k, grad[i], M, V, pin[i], has_target ? target[i] : T(0), has_target, PO, DL, acc);
    m[i] = M;
    v[i] = V;
    pout[i] = PO;
    if (delta) delta[i] = DL;
  }
  grid_reduce4<kThreads>(acc.partials(), partials, counter, [&](const ReducePartials& t) {
    sc->ssn = t.ssn;
    sc->changed = t.changed;
    sc->loss = has_target ? t.loss : nan("");
    sc->nonfinite = t.nonfinite;
    sc->ssn_used = ssn_in;
  });
}

// TMA-pipelined Adam update: grad, m, v, pi (+ target) streamed through a
// shared-memory ring by bulk copies, m, v, pi' stored from registers.
constexpr int kAdamArrays = 5;  // grad m v pin target

template <class T, bool FIRST, int kTh, int kSt, int kMinB>
__global__ void __launch_bounds__(kTh, kMinB)
    adam_update_tma_kernel(int64_t n, AdamK k, const T* grad, T* m, T* v, const T* pin, T* pout,
                           const T* target, T* delta, mg_update_scalars* sc,
                           ReducePartials* partials, unsigned int* counter) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kSt];
  constexpr int W = VecOf<T>::width;
  constexpr int TILE = kTh * W;
  T* sbuf = reinterpret_cast<T*>(smem_raw);
  const double ssn_in = __ldcg(&sc->ssn);
  const bool has_target = target != nullptr;
  const T* src[kAdamArrays] = {grad, m, v, pin, target};
  const bool use[kAdamArrays] = {true, !FIRST, !FIRST, true, has_target};
  uint32_t tx = 0;
#pragma unroll
  for (int a = 0; a < kAdamArrays; ++a) tx += use[a] ? uint32_t(TILE * sizeof(T)) : 0u;
  const int64_t tiles = n / TILE;
  const int64_t my_tiles =
      int64_t(blockIdx.x) < tiles ? (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kSt; ++st) mbar_init(&full[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = l2_evict_first_policy();
  auto issue = [&](int64_t li) {
    const int st = int(li % kSt);
    const int64_t tile = int64_t(blockIdx.x) + li * gridDim.x;
    mbar_arrive_expect_tx(&full[st], tx);
#pragma unroll
    for (int a = 0; a < kAdamArrays; ++a)
      if (use[a])
        bulk_g2s_hint(sbuf + (size_t(st) * kAdamArrays + a) * TILE, src[a] + tile * TILE,
                      uint32_t(TILE * sizeof(T)), &full[st], pol);
  };
  if (threadIdx.x == 0)
    for (int64_t li = 0; li < my_tiles && li < kSt; ++li) issue(li);
  Acc acc;
  const int e = threadIdx.x * W;
  for (int64_t li = 0; li < my_tiles; ++li) {
    const int st = int(li % kSt);
    mbar_wait(&full[st], uint32_t((li / kSt) & 1));
    const T* sb = sbuf + size_t(st) * kAdamArrays * TILE + e;
    const Pack<T> G = ld_plain(sb);
    Pack<T> M{}, V{}, TG{}, PO, DL;
    if (!FIRST) {
      M = ld_plain(sb + TILE);
      V = ld_plain(sb + 2 * TILE);
    }
    const Pack<T> PI = ld_plain(sb + 3 * TILE);
    if (has_target) TG = ld_plain(sb + 4 * TILE);
#pragma unroll
    for (int w = 0; w < W; ++w)
      adam_elem<T>(k, G.v[w], M.v[w], V.v[w], PI.v[w], TG.v[w], has_target, PO.v[w], DL.v[w],
                   acc);
    const int64_t b = (int64_t(blockIdx.x) + li * gridDim.x) * TILE + e;
    st_stream(m + b, M);
    st_stream(v + b, V);
    st_stream(pout + b, PO);
    if (delta) st_stream(delta + b, DL);
    __syncthreads();
    if (threadIdx.x == 0 && li + kSt < my_tiles) {
      fence_proxy_async_smem();
      issue(li + kSt);
    }
  }
  const int64_t tid = int64_t(blockIdx.x) * kTh + threadIdx.x;
  for (int64_t i = tiles * TILE + tid; i < n; i += int64_t(gridDim.x) * kTh) {
    T M = FIRST ? T(0) : m[i], V = FIRST ? T(0) : v[i], PO, DL;
    adam_elem<T>(k, grad[i], M, V, pin[i], has_target ? target[i] : T(0), has_target, PO, DL,
                 acc);
    m[i] = M;
    v[i] = V;
    pout[i] = PO;
    if (delta) delta[i] = DL;
  }
  grid_reduce4<kTh>(acc.partials(), partials, counter, [&](const ReducePartials& t) {
    sc->ssn = t.ssn;
    sc->changed = t.changed;
    sc->loss = has_target ? t.loss : nan("");
    sc->nonfinite = t.nonfinite;
    sc->ssn_used = ssn_in;
  });
}

// ------------------------------------------------------- standalone steps
template <class T>
__global__ void moment2_kernel(int64_t n, double c, bool first, T* __restrict__ m2,
                               const T* __restrict__ x) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const T old = first ? T(0) : m2[i];
    const T xi = x[i];
    m2[i] = old + T(c) * (xi * xi - old);  // moment2.hpp:38
  }
}

template <class T>
__global__ void negvar_check_kernel(int64_t n, const T* __restrict__ a, const T* __restrict__ b,
                                    int* flag) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    if (a[i] < T(0) || b[i] < T(0)) *flag = 1;  // meta.hpp:100
}

template <class T>
__global__ void meta_step_kernel(int64_t n, MetaK k, bool first, T* __restrict__ mean,
                                 T* __restrict__ var, T* __restrict__ ap,
                                 const T* __restrict__ prop, const T* __restrict__ diff,
                                 const T* __restrict__ vp, const T* __restrict__ vd,
                                 T* __restrict__ delta) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    T m = (first ? T(0) : mean[i]) + diff[i];
    T v = (first ? T(0) : var[i]) + vd[i];
    const T a_prev = first ? T(-INFINITY) : ap[i];
    const T vpi = vp[i];
    T al = div_z(vpi, (vpi + v) + T(k.eps_alpha));
    if (k.clip) al = std_min(al, T(1) / (T(2) - a_prev));
    ap[i] = al;
    const T om = T(1) - al;
    m = al * m + om * prop[i];
    v = (al * al) * v + (om * om) * vpi;
    mean[i] = m;
    var[i] = v;
    delta[i] = div_z(T(-k.lr) * m, sqrt_z(v) + T(k.eps_step));
  }
}

// compute_alpha (meta.hpp:38-47): the standalone weight with var_meta and
// var_diff kept apart, summed left to right as in the reference expression.
template <class T>
__global__ void compute_alpha_kernel(int64_t n, double eps_alpha, const T* __restrict__ vp,
                                     const T* __restrict__ vm, const T* __restrict__ vd,
                                     const T* __restrict__ ap, T* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const T raw = div_z(vp[i], ((vp[i] + vm[i]) + vd[i]) + T(eps_alpha));
    out[i] = std_min(raw, T(1) / (T(2) - ap[i]));
  }
}

// out = x * s (rescale_diff_variance, meta.hpp:51-53) or x / s (the bias
// corrections of Adam::m_hat / v_hat, adam.hpp:43-44).
template <class T>
__global__ void scalar_op_kernel(int64_t n, double s, int op, const T* __restrict__ x,
                                 T* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = op == 0 ? x[i] * T(s) : x[i] / T(s);
}

template <class T>
__global__ void adam_step_kernel(int64_t n, AdamK k, bool first, T* __restrict__ m,
                                 T* __restrict__ v, const T* __restrict__ g,
                                 T* __restrict__ delta) {
  Acc dummy;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    T M = first ? T(0) : m[i], V = first ? T(0) : v[i], PO, DL;
    adam_elem<T>(k, g[i], M, V, T(0), T(0), false, PO, DL, dummy);
    m[i] = M;
    v[i] = V;
    if (delta) delta[i] = DL;
  }
}

template <class T>
int launch_meta_update(mg_ctx* ctx, int64_t n, const MetaK& k, const MetaPtrs<T>& q, bool first,
                       mg_update_scalars* sc) {
  const bool vec = aligned16(q.prop) && aligned16(q.diff) && aligned16(q.m2p) &&
                   aligned16(q.m2d) && aligned16(q.mean) && aligned16(q.var) &&
                   aligned16(q.ap) && aligned16(q.pin) && aligned16(q.pout) &&
                   (!q.vprop || aligned16(q.vprop)) && (!q.vdiff || aligned16(q.vdiff)) &&
                   (!q.pprev || aligned16(q.pprev)) && (!q.target || aligned16(q.target)) &&
                   (!q.delta || aligned16(q.delta));
  const bool tma_ok = vec && !q.vprop && !q.vdiff && k.diff_norm == MG_DIFF_NORM_GLOBAL &&
                      n >= int64_t(tma_tile<T, 512>()) * ctx->sm_count && !g_disable_tma;
  if (tma_ok) {
    auto run_tma = [&](auto kernel, auto vc) {
      constexpr TmaVariant v = tma_variant(decltype(vc)::value);
      constexpr size_t smem = tma_smem_bytes<T, v.threads, v.stages>();
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      const int64_t tiles = n / tma_tile<T, v.threads>();
      const int64_t want = int64_t(ctx->sm_count) * v.ctas_per_sm;
      const int grid = int(tiles < want ? tiles : want);
      kernel<<<grid, v.threads, smem, ctx->stream>>>(n, k, q, sc, ctx->partials, ctx->counter);
    };
    auto pick = [&](auto vc) {
      constexpr TmaVariant v = tma_variant(decltype(vc)::value);
      if (first)
        run_tma(meta_update_tma_kernel<T, true, v.threads, v.stages, v.ctas_per_sm>, vc);
      else
        run_tma(meta_update_tma_kernel<T, false, v.threads, v.stages, v.ctas_per_sm>, vc);
    };
    // fp32: 640 threads x 2 stages from 2^26 parameters up (2^28: 2.24 ms
    // against 2.35 for 512 x 2), 512 x 2 below (2^24: 0.153 against
    // 0.167 ms, 2^25: 0.288 / 0.295; tools/update_variant_by_size.py)
    const int variant = g_tma_variant >= 0 ? g_tma_variant
                        : sizeof(T) == 4   ? (n >= (int64_t(3) << 24) ? 8 : 9)
                                           : 9;
    switch (variant) {
      case 1: pick(std::integral_constant<int, 1>{}); break;
      case 2: pick(std::integral_constant<int, 2>{}); break;
      case 3: pick(std::integral_constant<int, 3>{}); break;
      case 4: pick(std::integral_constant<int, 4>{}); break;
      case 5: pick(std::integral_constant<int, 5>{}); break;
      case 6: pick(std::integral_constant<int, 6>{}); break;
      case 7: pick(std::integral_constant<int, 7>{}); break;
      case 8: pick(std::integral_constant<int, 8>{}); break;
      case 9: pick(std::integral_constant<int, 9>{}); break;
      default: pick(std::integral_constant<int, 0>{}); break;
    }
    MG_LAUNCH_CHECK(ctx);
    return MG_OK;
  }
  const int64_t items = vec ? (n + VecOf<T>::width - 1) / VecOf<T>::width : n;
  const int grid = grid_for(ctx, items, kThreads, 8);
  auto run = [&](auto kernel) {
    kernel<<<grid, kThreads, 0, ctx->stream>>>(n, k, q, sc, ctx->partials, ctx->counter);
  };
  if (first)
    vec ? run(meta_update_kernel<T, true, true>) : run(meta_update_kernel<T, true, false>);
  else
    vec ? run(meta_update_kernel<T, false, true>) : run(meta_update_kernel<T, false, false>);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

template <class T>
int launch_adam_update(mg_ctx* ctx, int64_t n, const AdamK& k, bool first, const T* grad, T* m,
                       T* v, const T* pin, T* pout, const T* target, T* delta,
                       mg_update_scalars* sc) {
  const bool vec = aligned16(grad) && aligned16(m) && aligned16(v) && aligned16(pin) &&
                   aligned16(pout) && (!target || aligned16(target)) &&
                   (!delta || aligned16(delta));
  // TMA ring: MG_ADAM_THREADS threads x MG_ADAM_STAGES stages x 5 arrays per
  // CTA, MG_ADAM_CTAS CTAs/SM
  // (640 x 3 x 1: 1.19 ms at 2^28 fp32 against 1.29 for 192 x 4 x 2 and
  // 1.21-1.33 for 384-768 threads x 2-4 stages; tools/adam_probe.py)
#ifndef MG_ADAM_THREADS
#define MG_ADAM_THREADS 640
#define MG_ADAM_STAGES 3
#define MG_ADAM_CTAS 1
#endif
  constexpr int kTh = MG_ADAM_THREADS, kSt = MG_ADAM_STAGES;
  if (vec && !g_disable_tma && n >= int64_t(kTh) * VecOf<T>::width * ctx->sm_count) {
    constexpr size_t smem = size_t(kSt) * kAdamArrays * kTh * VecOf<T>::width * sizeof(T);
    auto run_tma = [&](auto kernel) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      const int64_t tiles = n / (int64_t(kTh) * VecOf<T>::width);
      const int64_t want = int64_t(ctx->sm_count) * MG_ADAM_CTAS;
      kernel<<<int(tiles < want ? tiles : want), kTh, smem, ctx->stream>>>(
          n, k, grad, m, v, pin, pout, target, delta, sc, ctx->partials, ctx->counter);
    };
    first ? run_tma(adam_update_tma_kernel<T, true, kTh, kSt, MG_ADAM_CTAS>)
          : run_tma(adam_update_tma_kernel<T, false, kTh, kSt, MG_ADAM_CTAS>);
    MG_LAUNCH_CHECK(ctx);
    return MG_OK;
  }
  const int64_t items = vec ? (n + VecOf<T>::width - 1) / VecOf<T>::width : n;
  const int grid = grid_for(ctx, items, kThreads, 8);
  auto run = [&](auto kernel) {
    kernel<<<grid, kThreads, 0, ctx->stream>>>(n, k, grad, m, v, pin, pout, target, delta, sc,
                                                ctx->partials, ctx->counter);
  };
  if (first)
    vec ? run(adam_update_kernel<T, true, true>) : run(adam_update_kernel<T, true, false>);
  else
    vec ? run(adam_update_kernel<T, false, true>) : run(adam_update_kernel<T, false, false>);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

MetaK make_meta_k(const mg_meta_update_args* a) {
  MetaK k;
  k.lr = a->meta.lr;
  k.eps_step = a->meta.eps_step;
  k.eps_alpha = a->meta.eps_alpha;
  k.clip = a->meta.clip_enabled;
  k.prop_coef = a->prop_coef;
  k.beta_f = a->beta_f;
  k.prop_dev = a->prop_coef_device;
  k.prop_adv = a->prop_pow_advance;
  k.beta_delta = a->beta_delta;
  k.diff_norm = a->diff_norm;
  k.project = a->project;
  k.proj_lo = a->proj_lo;
  k.proj_hi = a->proj_hi;
  k.ssn_from_host = a->ssn_from_host;
  k.ssn_host = a->ssn_host;
  return k;
}

// Advances the host-side Adam scalars exactly as adam.hpp:29-31 and returns
// the kernel constants.
AdamK advance_adam(mg_adam_scalars* s, int project, double proj_lo) {
  s->t += 1;
  s->beta1_pow *= s->beta1;
  s->beta2_pow *= s->beta2;
  AdamK k;
  k.beta1 = s->beta1;
  k.beta2 = s->beta2;
  k.c1 = 1.0 - s->beta1;
  k.c2 = 1.0 - s->beta2;
  k.d1 = 1.0 - s->beta1_pow;
  k.d2 = 1.0 - s->beta2_pow;
  k.lr = s->lr;
  k.eps = s->eps;
  k.project = project;
  k.proj_lo = proj_lo;
  return k;
}

// fp32: MG_FIX_* (default 512 texels x 5 channels per tile, one per thread,
// 2 stages of 102 KB, 1 CTA/SM: measured best of 9 shapes on configs[4],
// with 256 x 1 x 2 stages x 2 CTAs and 128 x 2 x 2 x 2 within 0.3 %);
// fp64: 128 texels, 3 stages (40 KB each), 1 CTA/SM
#ifndef MG_FIX_THREADS
#define MG_FIX_THREADS 512
#endif
#ifndef MG_FIX_TPT
#define MG_FIX_TPT 1
#endif
#ifndef MG_FIX_STAGES
#define MG_FIX_STAGES 2
#endif
#ifndef MG_FIX_MINB
#define MG_FIX_MINB 1
#endif
template <class T, int NCH>
struct FixShape {
  static constexpr int threads = sizeof(T) == 4 ? MG_FIX_THREADS : 128,
                       tpt = sizeof(T) == 4 ? MG_FIX_TPT : 1,
                       stages = sizeof(T) == 4 ? MG_FIX_STAGES : 3,
                       minb = sizeof(T) == 4 ? MG_FIX_MINB : 1;
  static constexpr int texels = threads * tpt;
};
template <class T, int NCH>
int launch_meta_update_fixed(mg_ctx* ctx, int64_t cells, int R2, const MetaK& k,
                             const MetaPtrs<T>& q, bool first, unsigned long long* acc,
                             unsigned int* touch, mg_update_scalars* sc) {
  using S = FixShape<T, NCH>;
  const int64_t n = cells * NCH;
  const bool tma_ok = !g_disable_tma && R2 % S::texels == 0 && k.diff_norm == MG_DIFF_NORM_GLOBAL &&
                      !q.target && !q.delta && aligned16(acc) && aligned16(q.m2p) &&
                      aligned16(q.m2d) && aligned16(q.mean) && aligned16(q.var) &&
                      aligned16(q.ap) && aligned16(q.pin) && (R2 * sizeof(T)) % 16 == 0 &&
                      cells / S::texels >= ctx->sm_count;
  if (tma_ok) {
    constexpr size_t smem = size_t(S::stages) * fix_stage_bytes<T, NCH, S::texels>();
    const int64_t tiles = cells / S::texels;
    const int64_t want = int64_t(ctx->sm_count) * S::minb;
    const int grid = int(tiles < want ? tiles : want);
    auto run = [&](auto kernel) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      kernel<<<grid, S::threads, smem, ctx->stream>>>(tiles, R2, k, q, acc, touch, sc,
                                                      ctx->partials, ctx->counter);
    };
    if constexpr (S::tpt == 1) {
      if (touch) {
        if (first)
          run(meta_update_fixed_tma_kernel<T, true, true, NCH, S::threads, S::tpt, S::stages,
                                           S::minb>);
        else
          run(meta_update_fixed_tma_kernel<T, false, true, NCH, S::threads, S::tpt, S::stages,
                                           S::minb>);
        MG_LAUNCH_CHECK(ctx);
        return MG_OK;
      }
    }
    // (a touch map with a multi-cell-per-thread shape: every cell is read
    // and zeroed, the map is left as it is - stale bits are harmless)
    if (first)
      run(meta_update_fixed_tma_kernel<T, true, false, NCH, S::threads, S::tpt, S::stages,
                                       S::minb>);
    else
      run(meta_update_fixed_tma_kernel<T, false, false, NCH, S::threads, S::tpt, S::stages,
                                       S::minb>);
  } else {
    const int grid = grid_for(ctx, n, kThreads, 8);
    auto run = [&](auto kernel) {
      kernel<<<grid, kThreads, 0, ctx->stream>>>(n, NCH, R2, k, q, acc, sc, ctx->partials,
                                                 ctx->counter);
    };
    first ? run(meta_update_fixed_kernel<T, true>) : run(meta_update_fixed_kernel<T, false>);
  }
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}
}  // namespace
}  // namespace mg

using namespace mg;

extern "C" {

int mg_set_option(const char* name, int64_t value) {
  if (!name) return fail(MG_EINVAL, "mg_set_option: null name");
  if (std::string(name) == "disable_tma") {
    g_disable_tma = value != 0;
    return MG_OK;
  }
  if (std::string(name) == "bvh_leaf_size") {
    if (value < 1 || value > 7) return fail(MG_EINVAL, "bvh_leaf_size must lie in [1, 7]");
    g_bvh_leaf = int(value);
    return MG_OK;
  }
  if (std::string(name) == "bvh_sah_axes") {
    if (value != 1 && value != 3) return fail(MG_EINVAL, "bvh_sah_axes must be 1 or 3");
    g_bvh_axes = int(value);
    return MG_OK;
  }
  if (std::string(name) == "bvh_bins") {
    if (value < 2 || value > 64) return fail(MG_EINVAL, "bvh_bins must lie in [2, 64]");
    g_bvh_bins = int(value);
    return MG_OK;
  }
  if (std::string(name) == "helix_split") {
    g_helix_split = value != 0;
    return MG_OK;
  }
  if (std::string(name) == "mesh_qnodes") {
    g_mesh_qnodes = value != 0;
    return MG_OK;
  }
  if (std::string(name) == "mesh_smem_stack") {
    g_mesh_smem_stack = value != 0;
    return MG_OK;
  }
  if (std::string(name) == "mesh_bvh8") {
    g_mesh_bvh8 = value != 0;
    return MG_OK;
  }
  if (std::string(name) == "mesh_scatter_aggregate") {
    g_mesh_scatter_agg = value != 0;
    return MG_OK;
  }
  if (std::string(name) == "mesh_persistent") {
    if (value < -1 || value > 3) return fail(MG_EINVAL, "mesh_persistent must lie in [-1, 3]");
    g_mesh_persistent = int(value);
    return MG_OK;
  }
  if (std::string(name) == "mesh_tail") {
    if (value < -1 || value > 8) return fail(MG_EINVAL, "mesh_tail must lie in [-1, 8]");
    g_mesh_tail = int(value);
    return MG_OK;
  }
  if (std::string(name) == "mesh_megakernel") {
    g_mesh_megakernel = value != 0;
    return MG_OK;
  }
  if (std::string(name) == "render_vec") {
    g_render_vec = value != 0;
    return MG_OK;
  }
  if (std::string(name) == "pool_keep_bytes") {
    if (value < 0) return fail(MG_EINVAL, "pool_keep_bytes must be non-negative");
    g_pool_keep = uint64_t(value);
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) apply_pool_keep(dev);
    return MG_OK;
  }
  if (std::string(name) == "cluster_runner") {
    g_cluster_runner = value != 0;
    return MG_OK;
  }
  if (std::string(name) == "render_fast") {
    g_render_fast = value != 0;
    return MG_OK;
  }
  if (std::string(name) == "render_fast_variant") {
    if (value < -1 || value >= render_fast_variants())
      return fail(MG_EINVAL, "render_fast_variant out of range");
    g_render_fast_variant = int(value);
    return MG_OK;
  }
  if (std::string(name) == "tma_variant") {
    if (value < -1 || value >= kNumTmaVariants) return fail(MG_EINVAL, "tma_variant out of range");
    g_tma_variant = int(value);
    return MG_OK;
  }
  return fail(MG_EINVAL, std::string("mg_set_option: unknown option ") + name);
}

int mg_meta_update(mg_ctx* ctx, int32_t dtype, int64_t n, const mg_meta_update_args* a,
                   const void* prop, const void* diff, void* m2_prop, void* m2_diff, void* mean,
                   void* var, void* alpha_prev, const void* params_in, void* params_out,
                   mg_update_scalars* scalars, const mg_meta_extras* x) {
  MG_NVTX("mg_meta_update");
  if (!ctx || !a || !scalars) return fail(MG_EINVAL, "mg_meta_update: null argument");
  if (n < 0) return fail(MG_EINVAL, "mg_meta_update: negative dimension");
  if (n == 0) return MG_OK;
  if (!prop || !diff || !m2_prop || !m2_diff || !mean || !var || !alpha_prev || !params_in ||
      !params_out)
    return fail(MG_EINVAL, "mg_meta_update: null buffer");
  if (a->diff_norm == MG_DIFF_NORM_PER_PARAM && !(x && x->params_prev))
    return fail(MG_EINVAL, "mg_meta_update: per-param diff norm needs params_prev");
  if (!(a->meta.lr > 0.0)) return fail(MG_EINVAL, "MetaEstimator: lr must be positive");
  if (a->prop_coef_device && !(a->beta_f > 0.0) && !a->prop_pow_advance)
    return fail(MG_EINVAL, "mg_meta_update: prop_coef_device with beta_f = 0 needs prop_pow_advance");
  const MetaK k = make_meta_k(a);
  const mg_meta_extras none{};
  const mg_meta_extras& e = x ? *x : none;
  if (dtype == MG_F32) {
    MetaPtrs<float> q{(const float*)prop, (const float*)diff, (const float*)e.vprop,
                      (const float*)e.vdiff, (float*)m2_prop, (float*)m2_diff, (float*)mean,
                      (float*)var, (float*)alpha_prev, (const float*)params_in,
                      (float*)params_out, (const float*)e.params_prev, (const float*)e.target,
                      (float*)e.delta_out};
    return launch_meta_update<float>(ctx, n, k, q, a->first_step != 0, scalars);
  }
  if (dtype == MG_F64) {
    MetaPtrs<double> q{(const double*)prop, (const double*)diff, (const double*)e.vprop,
                       (const double*)e.vdiff, (double*)m2_prop, (double*)m2_diff, (double*)mean,
                       (double*)var, (double*)alpha_prev, (const double*)params_in,
                       (double*)params_out, (const double*)e.params_prev,
                       (const double*)e.target, (double*)e.delta_out};
    return launch_meta_update<double>(ctx, n, k, q, a->first_step != 0, scalars);
  }
  return fail(MG_EINVAL, "mg_meta_update: unknown dtype");
}

// mg_meta_update with the sample pair in a texel-interleaved fixed-point
// accumulator (see meta_update_fixed_tma_kernel); the accumulator is zeroed.
int mg_meta_update_fixed(mg_ctx* ctx, int32_t dtype, int64_t cells, int32_t nch, int32_t r2,
                         const mg_meta_update_args* a, void* accum, void* m2_prop, void* m2_diff,
                         void* mean, void* var, void* alpha_prev, const void* params_in,
                         void* params_out, mg_update_scalars* scalars, const mg_meta_extras* x) {
  return mg_meta_update_fixed_touch(ctx, dtype, cells, nch, r2, a, accum, nullptr, m2_prop,
                                    m2_diff, mean, var, alpha_prev, params_in, params_out, scalars,
                                    x);
}

// touch_map (optional): bit c is set whenever cell c of accum may be
// non-zero; only those cells are read and zeroed, and their bits cleared.
int mg_meta_update_fixed_touch(mg_ctx* ctx, int32_t dtype, int64_t cells, int32_t nch, int32_t r2,
                               const mg_meta_update_args* a, void* accum, uint32_t* touch_map,
                               void* m2_prop, void* m2_diff, void* mean, void* var,
                               void* alpha_prev, const void* params_in, void* params_out,
                               mg_update_scalars* scalars, const mg_meta_extras* x) {
  MG_NVTX("mg_meta_update_fixed");
  if (!ctx || !a || !scalars) return fail(MG_EINVAL, "mg_meta_update_fixed: null argument");
  if (cells < 0 || r2 < 1 || (nch != 4 && nch != 5) || cells % r2 != 0)
    return fail(MG_EINVAL, "mg_meta_update_fixed: cells must be a multiple of r2 >= 1, nch 4 or 5");
  if (cells == 0) return MG_OK;
  if (!accum || !m2_prop || !m2_diff || !mean || !var || !alpha_prev || !params_in || !params_out)
    return fail(MG_EINVAL, "mg_meta_update_fixed: null buffer");
  if (x && (x->vprop || x->vdiff))
    return fail(MG_EUNSUPPORTED, "mg_meta_update_fixed: no independent variance pair");
  if (a->diff_norm == MG_DIFF_NORM_PER_PARAM && !(x && x->params_prev))
    return fail(MG_EINVAL, "mg_meta_update_fixed: per-param diff norm needs params_prev");
  if (!(a->meta.lr > 0.0)) return fail(MG_EINVAL, "MetaEstimator: lr must be positive");
  if (a->prop_coef_device && !(a->beta_f > 0.0) && !a->prop_pow_advance)
    return fail(MG_EINVAL, "mg_meta_update_fixed: prop_coef_device with beta_f = 0 needs prop_pow_advance");
  const MetaK k = make_meta_k(a);
  const mg_meta_extras none{};
  const mg_meta_extras& e = x ? *x : none;
  auto* acc = static_cast<unsigned long long*>(accum);
  auto go = [&](auto tag) {
    using T = decltype(tag);
    MetaPtrs<T> q{nullptr, nullptr, nullptr, nullptr, (T*)m2_prop, (T*)m2_diff, (T*)mean,
                  (T*)var, (T*)alpha_prev, (const T*)params_in, (T*)params_out,
                  (const T*)e.params_prev, (const T*)e.target, (T*)e.delta_out};
    return nch == 5 ? launch_meta_update_fixed<T, 5>(ctx, cells, r2, k, q, a->first_step != 0, acc,
                                                     touch_map, scalars)
                    : launch_meta_update_fixed<T, 4>(ctx, cells, r2, k, q, a->first_step != 0, acc,
                                                     touch_map, scalars);
  };
  if (dtype == MG_F32) return go(float{});
  if (dtype == MG_F64) return go(double{});
  return fail(MG_EINVAL, "mg_meta_update_fixed: unknown dtype");
}

int mg_shared_meta_update(mg_ctx* ctx, int32_t dtype, int64_t shard_n, int64_t shard_lo,
                          int32_t world, const mg_meta_update_args* a,
                          const void* const* prop_parts, const void* const* diff_parts,
                          void* const* params_out, const void* params_in, void* m2_prop,
                          void* m2_diff, void* mean, void* var, void* alpha_prev,
                          const void* target, mg_update_scalars* scalars) {
  if (!ctx || !a || !scalars || !prop_parts || !diff_parts || !params_out || !params_in)
    return fail(MG_EINVAL, "mg_shared_meta_update: null argument");
  if (world < 1 || world > kMaxPeers)
    return fail(MG_EINVAL, "mg_shared_meta_update: world must be 1..8");
  if (shard_n < 0 || shard_lo < 0) return fail(MG_EINVAL, "mg_shared_meta_update: bad shard");
  if (a->diff_norm != MG_DIFF_NORM_GLOBAL)
    return fail(MG_EUNSUPPORTED, "mg_shared_meta_update: global diff norm only");
  if (shard_n == 0) return MG_OK;
  if (a->prop_coef_device && !(a->beta_f > 0.0) && !a->prop_pow_advance)
    return fail(MG_EINVAL, "mg_shared_meta_update: prop_coef_device with beta_f = 0 needs prop_pow_advance");
  const MetaK k = make_meta_k(a);
  const bool first = a->first_step != 0;
  const int grid = grid_for(ctx, shard_n, kThreads, 8);
  auto go = [&](auto tag) {
    using T = decltype(tag);
    PeerPtrs<T> pp{};
    for (int q = 0; q < world; ++q) {
      pp.prop[q] = static_cast<const T*>(prop_parts[q]);
      pp.diff[q] = static_cast<const T*>(diff_parts[q]);
      pp.params_out[q] = static_cast<T*>(params_out[q]);
    }
    auto kern = first ? shared_meta_update_kernel<T, true> : shared_meta_update_kernel<T, false>;
    kern<<<grid, kThreads, 0, ctx->stream>>>(shard_n, shard_lo, world, k, pp,
                                             static_cast<const T*>(params_in),
                                             static_cast<T*>(m2_prop), static_cast<T*>(m2_diff),
                                             static_cast<T*>(mean), static_cast<T*>(var),
                                             static_cast<T*>(alpha_prev),
                                             static_cast<const T*>(target), scalars,
                                             ctx->partials, ctx->counter);
  };
  if (dtype == MG_F32)
    go(float{});
  else if (dtype == MG_F64)
    go(double{});
  else
    return fail(MG_EINVAL, "mg_shared_meta_update: unknown dtype");
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

int mg_adam_update(mg_ctx* ctx, int32_t dtype, int64_t n, mg_adam_scalars* s, int32_t project,
                   double proj_lo, const void* grad, void* m, void* v, const void* params_in,
                   void* params_out, const void* target, mg_update_scalars* scalars) {
  MG_NVTX("mg_adam_update");
  if (!ctx || !s || !scalars) return fail(MG_EINVAL, "mg_adam_update: null argument");
  if (n < 0) return fail(MG_EINVAL, "mg_adam_update: negative dimension");
  if (n == 0) return MG_OK;
  const bool first = s->t == 0;
  const AdamK k = advance_adam(s, project, proj_lo);
  if (dtype == MG_F32)
    return launch_adam_update<float>(ctx, n, k, first, (const float*)grad, (float*)m, (float*)v,
                                     (const float*)params_in, (float*)params_out,
                                     (const float*)target, nullptr, scalars);
  if (dtype == MG_F64)
    return launch_adam_update<double>(ctx, n, k, first, (const double*)grad, (double*)m,
                                      (double*)v, (const double*)params_in, (double*)params_out,
                                      (const double*)target, nullptr, scalars);
  return fail(MG_EINVAL, "mg_adam_update: unknown dtype");
}

int mg_moment2_step(mg_ctx* ctx, int32_t dtype, int64_t n, mg_moment2_scalars* s, void* m2,
                    const void* x) {
  if (!ctx || !s) return fail(MG_EINVAL, "mg_moment2_step: null argument");
  if (!(s->decay >= 0.0 && s->decay < 1.0))
    return fail(MG_EINVAL, "Moment2: decay must lie in [0, 1)");
  const bool first = s->count == 0;
  s->count += 1;                      // moment2.hpp:34
  s->decay_pow *= s->decay;           // moment2.hpp:35
  const double w = 1.0 - s->decay;    // moment2.hpp:36
  const double w_sum = 1.0 - s->decay_pow;
  const double c = w / w_sum;
  if (n == 0) return MG_OK;
  const int grid = grid_for(ctx, n, 256, 8);
  if (dtype == MG_F32)
    moment2_kernel<float><<<grid, 256, 0, ctx->stream>>>(n, c, first, (float*)m2, (const float*)x);
  else if (dtype == MG_F64)
    moment2_kernel<double><<<grid, 256, 0, ctx->stream>>>(n, c, first, (double*)m2,
                                                          (const double*)x);
  else
    return fail(MG_EINVAL, "mg_moment2_step: unknown dtype");
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

int mg_meta_step(mg_ctx* ctx, int32_t dtype, int64_t n, const mg_meta_params* p,
                 int32_t first_call, void* mean, void* var, void* alpha_prev, const void* prop,
                 const void* diff, const void* var_prop, const void* var_diff, void* delta) {
  if (!ctx || !p) return fail(MG_EINVAL, "mg_meta_step: null argument");
  if (!(p->lr > 0.0)) return fail(MG_EINVAL, "MetaEstimator: lr must be positive");
  if (n == 0) return MG_OK;
  if (dtype != MG_F32 && dtype != MG_F64) return fail(MG_EINVAL, "mg_meta_step: unknown dtype");
  const int grid = grid_for(ctx, n, 256, 8);
  MG_CUDA_TRY(cudaMemsetAsync(ctx->flag, 0, sizeof(int), ctx->stream));
  if (dtype == MG_F32)
    negvar_check_kernel<float><<<grid, 256, 0, ctx->stream>>>(n, (const float*)var_prop,
                                                              (const float*)var_diff, ctx->flag);
  else
    negvar_check_kernel<double><<<grid, 256, 0, ctx->stream>>>(n, (const double*)var_prop,
                                                               (const double*)var_diff, ctx->flag);
  MG_LAUNCH_CHECK(ctx);
  int flag = 0;
  MG_CUDA_TRY(cudaMemcpyAsync(&flag, ctx->flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (flag) return fail(MG_ELOGIC, "MetaEstimator: negative variance input");
  MetaK k{};
  k.lr = p->lr;
  k.eps_step = p->eps_step;
  k.eps_alpha = p->eps_alpha;
  k.clip = p->clip_enabled;
  if (dtype == MG_F32)
    meta_step_kernel<float><<<grid, 256, 0, ctx->stream>>>(
        n, k, first_call != 0, (float*)mean, (float*)var, (float*)alpha_prev, (const float*)prop,
        (const float*)diff, (const float*)var_prop, (const float*)var_diff, (float*)delta);
  else
    meta_step_kernel<double><<<grid, 256, 0, ctx->stream>>>(
        n, k, first_call != 0, (double*)mean, (double*)var, (double*)alpha_prev,
        (const double*)prop, (const double*)diff, (const double*)var_prop,
        (const double*)var_diff, (double*)delta);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

int mg_adam_step(mg_ctx* ctx, int32_t dtype, int64_t n, mg_adam_scalars* s, void* m, void* v,
                 const void* grad, void* delta) {
  if (!ctx || !s) return fail(MG_EINVAL, "mg_adam_step: null argument");
  if (!(s->lr > 0.0)) return fail(MG_EINVAL, "Adam: lr must be positive");
  if (!(s->beta1 >= 0.0 && s->beta1 < 1.0) || !(s->beta2 >= 0.0 && s->beta2 < 1.0))
    return fail(MG_EINVAL, "Adam: betas must lie in [0, 1)");
  const bool first = s->t == 0;
  const AdamK k = advance_adam(s, 0, 0.0);
  if (n == 0) return MG_OK;
  const int grid = grid_for(ctx, n, 256, 8);
  if (dtype == MG_F32)
    adam_step_kernel<float><<<grid, 256, 0, ctx->stream>>>(n, k, first, (float*)m, (float*)v,
                                                           (const float*)grad, (float*)delta);
  else if (dtype == MG_F64)
    adam_step_kernel<double><<<grid, 256, 0, ctx->stream>>>(n, k, first, (double*)m, (double*)v,
                                                            (const double*)grad, (double*)delta);
  else
    return fail(MG_EINVAL, "mg_adam_step: unknown dtype");
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

int mg_compute_alpha(mg_ctx* ctx, int32_t dtype, int64_t n, const void* var_prop,
                     const void* var_meta, const void* var_diff, const void* alpha_prev,
                     double eps_alpha, void* out) {
  if (!ctx) return fail(MG_EINVAL, "mg_compute_alpha: null argument");
  if (n < 0) return fail(MG_EINVAL, "compute_alpha: dimension mismatch");
  if (n == 0) return MG_OK;
  if (!var_prop || !var_meta || !var_diff || !alpha_prev || !out)
    return fail(MG_EINVAL, "mg_compute_alpha: null argument");
  if (dtype != MG_F32 && dtype != MG_F64) return fail(MG_EINVAL, "mg_compute_alpha: unknown dtype");
  const int grid = grid_for(ctx, n, 256, 8);
  MG_CUDA_TRY(cudaMemsetAsync(ctx->flag, 0, sizeof(int), ctx->stream));
  if (dtype == MG_F32) {
    negvar_check_kernel<float><<<grid, 256, 0, ctx->stream>>>(n, (const float*)var_prop,
                                                              (const float*)var_meta, ctx->flag);
    negvar_check_kernel<float><<<grid, 256, 0, ctx->stream>>>(n, (const float*)var_diff,
                                                              (const float*)var_diff, ctx->flag);
  } else {
    negvar_check_kernel<double><<<grid, 256, 0, ctx->stream>>>(n, (const double*)var_prop,
                                                               (const double*)var_meta, ctx->flag);
    negvar_check_kernel<double><<<grid, 256, 0, ctx->stream>>>(n, (const double*)var_diff,
                                                               (const double*)var_diff, ctx->flag);
  }
  MG_LAUNCH_CHECK(ctx);
  ctx->launches++;
  int flag = 0;
  MG_CUDA_TRY(cudaMemcpyAsync(&flag, ctx->flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (flag) return fail(MG_ELOGIC, "compute_alpha: negative variance input");
  if (dtype == MG_F32)
    compute_alpha_kernel<float><<<grid, 256, 0, ctx->stream>>>(
        n, eps_alpha, (const float*)var_prop, (const float*)var_meta, (const float*)var_diff,
        (const float*)alpha_prev, (float*)out);
  else
    compute_alpha_kernel<double><<<grid, 256, 0, ctx->stream>>>(
        n, eps_alpha, (const double*)var_prop, (const double*)var_meta, (const double*)var_diff,
        (const double*)alpha_prev, (double*)out);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

int mg_scalar_op(mg_ctx* ctx, int32_t dtype, int64_t n, const void* x, double s, int32_t op,
                 void* out) {
  if (!ctx || (n > 0 && (!x || !out))) return fail(MG_EINVAL, "mg_scalar_op: null argument");
  if (op != 0 && op != 1) return fail(MG_EINVAL, "mg_scalar_op: op must be 0 (mul) or 1 (div)");
  if (n <= 0) return n < 0 ? fail(MG_EINVAL, "mg_scalar_op: negative size") : MG_OK;
  const int grid = grid_for(ctx, n, 256, 8);
  if (dtype == MG_F32)
    scalar_op_kernel<float><<<grid, 256, 0, ctx->stream>>>(n, s, op, (const float*)x, (float*)out);
  else if (dtype == MG_F64)
    scalar_op_kernel<double><<<grid, 256, 0, ctx->stream>>>(n, s, op, (const double*)x,
                                                            (double*)out);
  else
    return fail(MG_EINVAL, "mg_scalar_op: unknown dtype");
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

}  // extern "C"
