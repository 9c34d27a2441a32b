// Shared device/host plumbing for libmgcuda (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include <nvtx3/nvToolsExt.h>

#include "mgcuda.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libmgcuda targets sm_100a (B200) only"
#endif

namespace mg {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define MG_CUDA_TRY(expr)                                  \
  do {                                                     \
    cudaError_t mg_e_ = (expr);                            \
    if (mg_e_ != cudaSuccess) return ::mg::cuda_fail(mg_e_, #expr); \
  } while (0)

#define MG_LAUNCH_CHECK(ctx)                               \
  do {                                                     \
    (ctx)->launches++;                                     \
    cudaError_t mg_e_ = cudaGetLastError();                \
    if (mg_e_ != cudaSuccess) return ::mg::cuda_fail(mg_e_, "kernel launch"); \
  } while (0)

// Device-side invariant checks, compiled in only for the debug-check build
// (make -C paper_2309_15676_b200/csrc debug -> libmgcuda_debug.so, used by
// tools/debug_checks.sh in place of compute-sanitizer, which is closed on
// the GPU pool): ring / tile bounds, queue and stack capacities,
// accumulator cells, reduction grid sizes.  A failed check is a device
// assert (message + trap).
#ifdef MG_DEBUG_CHECKS
#include <assert.h>
#define MG_DCHECK(x) assert(x)
#else
#define MG_DCHECK(x) ((void)0)
#endif

// NVTX range over a host entry point / pipeline stage (header-only NVTX3: a
// no-op unless a profiler injects itself; ncu --nvtx --nvtx-include can
// filter kernels by these names)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define MG_NVTX_CAT2(a, b) a##b
#define MG_NVTX_CAT(a, b) MG_NVTX_CAT2(a, b)
#define MG_NVTX(name) ::mg::NvtxRange MG_NVTX_CAT(mg_nvtx_, __LINE__)(name)

// across-replicate aggregation (aggregate.cu); runs[r * runs_stride] are the
// replicates' iterations_run
int launch_aggregate(mg_ctx* ctx, int S, int R, int T, const double* series, const int32_t* runs,
                     int runs_stride, double* stats, int32_t* active);

// ----------------------------------------------------------------- context
// Reduction epilogue workspace: per-block partials + arrival counter.
constexpr int kMaxReduceBlocks = 148 * 16;
struct ReducePartials {
  double ssn, changed, loss, nonfinite;
};
// Per-thread accumulators of the fused epilogue (counts kept as integers).
struct Acc {
  double ssn = 0.0, loss = 0.0;
  unsigned int changed = 0, nonfinite = 0;
  __host__ __device__ ReducePartials partials() const {
    return ReducePartials{ssn, double(changed), loss, double(nonfinite)};
  }
};

}  // namespace mg

struct mg_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  bool owns_stream = false;
  int64_t launches = 0;
  // device workspace
  mg::ReducePartials* partials = nullptr;  // [kMaxReduceBlocks]
  unsigned int* counter = nullptr;         // arrival counter (self-resetting)
  int* flag = nullptr;                     // error flag for validation kernels
  // device iteration offset (mg_ctx_set_iteration_offset): sample-pair
  // kernels launched on this context use iteration + *it_offset
  const uint32_t* it_offset = nullptr;
  // work counter of dynamically scheduled kernels (zeroed before each use)
  unsigned int* work = nullptr;
  // grow-only scratch (mg::ctx_scratch); stream-ordered reuse by one call at
  // a time, like the reduction workspace
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
};

namespace mg {

// ------------------------------------------------- fixed-point accumulation
// Fire-and-forget 64-bit integer add into GLOBAL memory (RED: no value comes
// back).  atomicAdd on a pointer the compiler cannot prove global compiles
// to a generic-address ATOM with a return value plus a shared-window CAS
// branch; the adjoint scatters discard the result, so RED is the whole
// operation.  No "memory" clobber: nothing in a scattering kernel reads the
// accumulator, so independent loads may be scheduled across the adds.
// Integer adds commute: the sums are the same bits in any order.
__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v));
}

// --------------------------------------------------------------- dtype utils
template <class T>
struct VecOf;
template <>
struct VecOf<float> {
  using type = float4;
  static constexpr int width = 4;
};
template <>
struct VecOf<double> {
  using type = double2;
  static constexpr int width = 2;
};

// Streaming (evict-first) 128-bit load/store of VEC elements of T.
template <class T>
struct Pack {
  static constexpr int W = VecOf<T>::width;
  T v[W];
};

template <class T>
__device__ __forceinline__ Pack<T> ld_stream(const T* p) {
  Pack<T> r;
  auto x = __ldcs(reinterpret_cast<const typename VecOf<T>::type*>(p));
  static_assert(sizeof(x) == sizeof(r), "pack size");
  memcpy(&r, &x, sizeof(r));
  return r;
}

template <class T>
__device__ __forceinline__ Pack<T> ld_plain(const T* p) {
  Pack<T> r;
  auto x = *reinterpret_cast<const typename VecOf<T>::type*>(p);
  memcpy(&r, &x, sizeof(r));
  return r;
}

template <class T>
__device__ __forceinline__ void st_plain(T* p, const Pack<T>& r) {
  typename VecOf<T>::type x;
  memcpy(&x, &r, sizeof(r));
  *reinterpret_cast<typename VecOf<T>::type*>(p) = x;
}

template <class T>
__device__ __forceinline__ void st_stream(T* p, const Pack<T>& r) {
  typename VecOf<T>::type x;
  memcpy(&x, &r, sizeof(r));
  __stcs(reinterpret_cast<typename VecOf<T>::type*>(p), x);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// std::min / std::max semantics (Eigen numext::mini/maxi), NaN-faithful:
// min(a,b) = (b < a) ? b : a ; max(a,b) = (a < b) ? b : a
template <class T>
__device__ __forceinline__ T std_min(T a, T b) { return (b < a) ? b : a; }
template <class T>
__device__ __forceinline__ T std_max(T a, T b) { return (a < b) ? b : a; }

// ------------------------------------------------ deterministic reductions
// Fixed-shape tree over a block: warp shuffles then one warp over warp sums.
template <int kThreads>
__device__ __forceinline__ double block_sum(double v, double* smem_warp) {
  static_assert(kThreads % 32 == 0 && kThreads <= 1024, "block shape");
  constexpr int kWarps = kThreads / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) smem_warp[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = lane < kWarps ? smem_warp[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  return r;  // valid in thread 0
}

// Block partials -> ReducePartials[blockIdx]; the last block to arrive sums
// the partials in block order (deterministic) and calls fin(total) in
// thread 0.  Resets the counter for the next launch.
template <int kThreads, class Fin>
__device__ __forceinline__ void grid_reduce4(ReducePartials acc, ReducePartials* partials,
                                             unsigned int* counter, Fin fin) {
  __shared__ double sw[kThreads / 32];
  __shared__ bool is_last;
  MG_DCHECK(gridDim.x <= unsigned(kMaxReduceBlocks) && blockDim.x == unsigned(kThreads));
  const double s0 = block_sum<kThreads>(acc.ssn, sw);
  const double s1 = block_sum<kThreads>(acc.changed, sw);
  const double s2 = block_sum<kThreads>(acc.loss, sw);
  const double s3 = block_sum<kThreads>(acc.nonfinite, sw);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = ReducePartials{s0, s1, s2, s3};
    __threadfence();
    const unsigned int prev = atomicAdd(counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // Last block: each thread sums a strided subset in order, then the fixed tree.
  ReducePartials t{0.0, 0.0, 0.0, 0.0};
  for (unsigned int b = threadIdx.x; b < gridDim.x; b += kThreads) {
    const ReducePartials p = partials[b];
    t.ssn += p.ssn;
    t.changed += p.changed;
    t.loss += p.loss;
    t.nonfinite += p.nonfinite;
  }
  const double r0 = block_sum<kThreads>(t.ssn, sw);
  const double r1 = block_sum<kThreads>(t.changed, sw);
  const double r2 = block_sum<kThreads>(t.loss, sw);
  const double r3 = block_sum<kThreads>(t.nonfinite, sw);
  if (threadIdx.x == 0) {
    fin(ReducePartials{r0, r1, r2, r3});
    *counter = 0u;
  }
}

// The context's scratch with at least `bytes` (grown with a synchronising
// reallocation, so a size reached once is stable — e.g. across CUDA-graph
// capture of a loop whose first step ran eagerly); nullptr on failure.
inline void* ctx_scratch(mg_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->scratch_bytes) return ctx->scratch;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return nullptr;
  cudaFree(ctx->scratch);
  ctx->scratch = nullptr;
  ctx->scratch_bytes = 0;
  if (cudaMalloc(&ctx->scratch, bytes) != cudaSuccess) return nullptr;
  ctx->scratch_bytes = bytes;
  return ctx->scratch;
}

inline int grid_for(const mg_ctx* ctx, int64_t items, int threads, int blocks_per_sm) {
  int64_t g = (items + threads - 1) / threads;
  const int64_t cap = int64_t(ctx->sm_count) * blocks_per_sm;
  if (g > cap) g = cap;
  if (g > kMaxReduceBlocks) g = kMaxReduceBlocks;
  if (g < 1) g = 1;
  return int(g);
}

}  // namespace mg
