// Context, error plumbing and ExperimentConfig validation for libmgcuda.
#include <string.h>

#include <string>

#include "mg_common.cuh"

namespace mg {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return e == cudaErrorMemoryAllocation ? MG_ENOMEM : MG_ECUDA;
}

}  // namespace mg

using namespace mg;

namespace {
template <class T>
__global__ void fill_kernel(int64_t n, T* dst, T v) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = v;
}
}  // namespace

namespace mg {
// Bytes the device's default stream-ordered pool keeps mapped across
// synchronisations (cudaMemPoolAttrReleaseThreshold; the CUDA default is 0:
// every sync unmaps what was freed, so each runner call re-maps its
// workspace).  mg_set_option("pool_keep_bytes", n).
uint64_t g_pool_keep = uint64_t(512) << 20;

int apply_pool_keep(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return MG_ECUDA;
  uint64_t keep = g_pool_keep;
  return cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep) == cudaSuccess
             ? MG_OK
             : MG_ECUDA;
}
__global__ void counter_add_kernel(uint32_t* c, uint32_t inc) { *c += inc; }
}  // namespace mg

extern "C" {

int mg_fill(mg_ctx* ctx, int32_t dtype, int64_t n, void* dst, double value) {
  if (!ctx || (n && !dst)) return fail(MG_EINVAL, "mg_fill: null argument");
  if (n <= 0) return MG_OK;
  const int grid = grid_for(ctx, n, 256, 8);
  if (dtype == MG_F32)
    fill_kernel<float><<<grid, 256, 0, ctx->stream>>>(n, (float*)dst, float(value));
  else if (dtype == MG_F64)
    fill_kernel<double><<<grid, 256, 0, ctx->stream>>>(n, (double*)dst, value);
  else
    return fail(MG_EINVAL, "mg_fill: unknown dtype");
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

const char* mg_last_error(void) { return g_last_error.c_str(); }

int mg_abi_version(void) { return MGCUDA_ABI_VERSION; }

// Debug-check builds only: launches one kernel whose MG_DCHECK fails, so a
// harness can prove the checks are compiled in (the launch then reports
// the device assert as MG_ECUDA).  Release builds: MG_EUNSUPPORTED.
__global__ void mg_dcheck_selftest_kernel(int x) { MG_DCHECK(x == 0); }

int mg_debug_selftest(mg_ctx* ctx) {
#ifdef MG_DEBUG_CHECKS
  if (!ctx) return mg::fail(MG_EINVAL, "mg_debug_selftest: null context");
  mg_dcheck_selftest_kernel<<<1, 1, 0, ctx->stream>>>(1);
  MG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return MG_OK;
#else
  (void)ctx;
  return mg::fail(MG_EUNSUPPORTED, "mg_debug_selftest: release build (no device checks)");
#endif
}

// harness.hpp:18-67 field defaults
void mg_config_defaults(mg_experiment_config* c) {
  memset(c, 0, sizeof(*c));
  c->problem = MG_EXP_RATE;
  c->optimizer = MG_OPT_META;
  c->iterations = 100;
  c->replicates = 1;
  c->seed = 0;
  c->lr = 0.01;
  c->beta_f = 0.9;
  c->beta_delta = 0.5;
  c->beta1 = 0.9;
  c->beta2 = 0.999;
  c->eps_step = 1e-8;
  c->eps_alpha = 1e-30;
  c->adam_eps = 1e-8;
  c->dim = 4;
  c->sigma = 1.0;
  c->samples_per_iter = 32;
  c->target_mean = 2.0;
  c->rate_init = 2.0;
  c->pixel_count = 8;
  c->spp = 4;
  c->problem_seed = 1234;
  c->albedo_init = 0.1;
  c->exponent_max = 4.0;
  c->trajectory = MG_TRAJ_OPTIMISE;
  c->traj_rate = 0.05;
  c->diff_norm = MG_DIFF_NORM_GLOBAL;
  c->coord = 0;
  c->converge_threshold = -1.0;
  c->dtype = MG_F64;
  c->rng = MG_RNG_MT64;
}

// ExperimentConfig::validate (harness.cpp:42-66), same messages.
int mg_config_validate(const mg_experiment_config* c) {
  if (!c) return fail(MG_EINVAL, "null config");
  if (c->problem < 0 || c->problem > 2)
    return fail(MG_EINVAL, "unknown problem (valid: exp-rate, mult-noise, mini-render)");
  if (c->optimizer < 0 || c->optimizer > 1)
    return fail(MG_EINVAL, "unknown optimizer (valid: meta, adam)");
  if (c->trajectory < 0 || c->trajectory > 2)
    return fail(MG_EINVAL, "unknown trajectory (valid: optimise, scripted-linear, scripted-exp)");
  if (c->diff_norm < 0 || c->diff_norm > 1)
    return fail(MG_EINVAL, "unknown diff-norm (valid: global, per-param)");
  if (c->iterations < 1) return fail(MG_EINVAL, "iterations must be >= 1");
  if (c->replicates < 1) return fail(MG_EINVAL, "replicates must be >= 1");
  if (!(c->lr > 0.0)) return fail(MG_EINVAL, "lr must be positive");
  if (!(c->beta_f >= 0.0 && c->beta_f < 1.0)) return fail(MG_EINVAL, "beta-f must lie in [0, 1)");
  if (!(c->beta_delta >= 0.0 && c->beta_delta < 1.0))
    return fail(MG_EINVAL, "beta-delta must lie in [0, 1)");
  if (!(c->beta1 >= 0.0 && c->beta1 < 1.0)) return fail(MG_EINVAL, "beta1 must lie in [0, 1)");
  if (!(c->beta2 >= 0.0 && c->beta2 < 1.0)) return fail(MG_EINVAL, "beta2 must lie in [0, 1)");
  if (c->coord < 0) return fail(MG_EINVAL, "coord must be >= 0");
  if (c->non_zero_centred)
    return fail(MG_EINVAL,
                "non-zero-centred variance approximation is a reserved ablation and is not "
                "implemented");
  if (c->dtype != MG_F32 && c->dtype != MG_F64) return fail(MG_EINVAL, "dtype must be f32 or f64");
  if (c->rng != MG_RNG_MT64 && c->rng != MG_RNG_PHILOX)
    return fail(MG_EINVAL, "rng must be mt64 or philox");
  return MG_OK;
}

int mg_ctx_create(int device, void* stream, mg_ctx** out) {
  if (!out) return fail(MG_EINVAL, "mg_ctx_create: null out");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(MG_ECUDA, "no CUDA device visible: libmgcuda needs a B200 (sm_100a); there is "
                          "no CPU fallback");
  if (device < 0 || device >= count) return fail(MG_EINVAL, "mg_ctx_create: bad device index");
  cudaDeviceProp prop;
  MG_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0)
    return fail(MG_ECUDA, std::string("libmgcuda is built for sm_100a only; device is sm_") +
                              std::to_string(prop.major) + std::to_string(prop.minor));
  MG_CUDA_TRY(cudaSetDevice(device));
  apply_pool_keep(device);
  mg_ctx* ctx = new mg_ctx();
  ctx->device = device;
  ctx->sm_count = prop.multiProcessorCount;
  if (stream) {
    ctx->stream = static_cast<cudaStream_t>(stream);
  } else {
    e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete ctx;
      return cuda_fail(e, "cudaStreamCreate");
    }
    ctx->owns_stream = true;
  }
  e = cudaMalloc(&ctx->partials, sizeof(ReducePartials) * kMaxReduceBlocks);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->counter, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->flag, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&ctx->work, sizeof(unsigned int));
  // ordered on the context's stream (it may not synchronise with the legacy one)
  if (e == cudaSuccess) e = cudaMemsetAsync(ctx->counter, 0, sizeof(unsigned int), ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    mg_ctx_destroy(ctx);
    return cuda_fail(e, "mg_ctx_create workspace");
  }
  *out = ctx;
  return MG_OK;
}

int mg_ctx_destroy(mg_ctx* ctx) {
  if (!ctx) return MG_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  cudaFree(ctx->partials);
  cudaFree(ctx->counter);
  cudaFree(ctx->flag);
  cudaFree(ctx->work);
  cudaFree(ctx->scratch);
  if (ctx->owns_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return MG_OK;
}

int mg_ctx_synchronize(mg_ctx* ctx) {
  if (!ctx) return fail(MG_EINVAL, "null ctx");
  MG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return MG_OK;
}

void* mg_ctx_stream(mg_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int mg_ctx_set_iteration_offset(mg_ctx* ctx, const uint32_t* dev_counter) {
  if (!ctx) return fail(MG_EINVAL, "mg_ctx_set_iteration_offset: null context");
  ctx->it_offset = dev_counter;
  return MG_OK;
}

int mg_iteration_offset_add(mg_ctx* ctx, uint32_t* dev_counter, uint32_t inc) {
  if (!ctx || !dev_counter) return fail(MG_EINVAL, "mg_iteration_offset_add: null argument");
  mg::counter_add_kernel<<<1, 1, 0, ctx->stream>>>(dev_counter, inc);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

int64_t mg_ctx_launch_count(mg_ctx* ctx) { return ctx ? ctx->launches : 0; }

int mg_scalars_read(mg_ctx* ctx, const mg_update_scalars* dev, mg_update_scalars* host) {
  if (!ctx || !dev || !host) return fail(MG_EINVAL, "mg_scalars_read: null argument");
  MG_CUDA_TRY(cudaMemcpyAsync(host, dev, sizeof(*host), cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return MG_OK;
}

int mg_scalars_write(mg_ctx* ctx, mg_update_scalars* dev, const mg_update_scalars* host) {
  if (!ctx || !dev || !host) return fail(MG_EINVAL, "mg_scalars_write: null argument");
  MG_CUDA_TRY(cudaMemcpyAsync(dev, host, sizeof(*host), cudaMemcpyHostToDevice, ctx->stream));
  MG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return MG_OK;
}

int mg_malloc(mg_ctx* ctx, size_t bytes, void** out) {
  if (!ctx || !out) return fail(MG_EINVAL, "mg_malloc: null argument");
  *out = nullptr;
  if (bytes == 0) return MG_OK;
  MG_CUDA_TRY(cudaMallocAsync(out, bytes, ctx->stream));
  return MG_OK;
}

int mg_free(mg_ctx* ctx, void* p) {
  if (!ctx) return fail(MG_EINVAL, "mg_free: null ctx");
  if (p) MG_CUDA_TRY(cudaFreeAsync(p, ctx->stream));
  return MG_OK;
}

static int copy_sync(mg_ctx* ctx, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  if (!ctx || (bytes && (!dst || !src))) return fail(MG_EINVAL, "mg_copy: null argument");
  if (bytes == 0) return MG_OK;
  MG_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, kind, ctx->stream));
  MG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return MG_OK;
}

int mg_copy_to_device(mg_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return copy_sync(ctx, dst, src, bytes, cudaMemcpyHostToDevice);
}
int mg_copy_to_host(mg_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return copy_sync(ctx, dst, src, bytes, cudaMemcpyDeviceToHost);
}
int mg_copy_device(mg_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!ctx || (bytes && (!dst || !src))) return fail(MG_EINVAL, "mg_copy_device: null argument");
  if (bytes) MG_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  return MG_OK;
}

int mg_host_malloc(size_t bytes, void** out) {
  if (!out) return fail(MG_EINVAL, "mg_host_malloc: null argument");
  *out = nullptr;
  if (bytes == 0) return MG_OK;
  MG_CUDA_TRY(cudaMallocHost(out, bytes));
  return MG_OK;
}

int mg_host_free(void* p) {
  if (p) MG_CUDA_TRY(cudaFreeHost(p));
  return MG_OK;
}

int mg_copy_async(mg_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!ctx || (bytes && (!dst || !src))) return fail(MG_EINVAL, "mg_copy_async: null argument");
  if (bytes) MG_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
  return MG_OK;
}

uint64_t mg_mix64(uint64_t x) {
  // rng.hpp:9-14
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t mg_stream_seed(uint64_t base_seed, uint64_t replicate) {
  return mg_mix64(mg_mix64(base_seed) ^ (replicate + 0x51ed2701e35f3a6dULL));  // rng.hpp:23-25
}

}  // extern "C"
