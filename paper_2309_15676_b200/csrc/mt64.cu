// Batched device std::mt19937_64 engines (row A1, rng.hpp:18-37).
#include <vector>

#include "mg_common.cuh"
#include "mt64.cuh"
#include "mt64_state.h"

namespace mg {
namespace {

constexpr int kDrawThreads = 160;

__global__ void mt_seed_kernel(int streams, const uint64_t* __restrict__ seeds,
                               uint64_t* __restrict__ state, int* __restrict__ idx) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= streams) return;
  mt_seed(state + size_t(r) * kMtN, seeds[r]);
  idx[r] = kMtN;
}

// kind 0: raw, 1: uniform (rng.hpp:28), 2: uniform_pos (rng.hpp:31)
__global__ void __launch_bounds__(kDrawThreads)
    mt_draw_kernel(int64_t n, int kind, uint64_t* __restrict__ state, int* __restrict__ idx,
                   void* __restrict__ out) {
  __shared__ uint64_t sbuf[2][kMtN];
  const int r = blockIdx.x;
  MtBlock e{{sbuf[0], sbuf[1]}, 0, 0};
  mt_block_load(e, state + size_t(r) * kMtN, idx[r]);
  uint64_t* o64 = static_cast<uint64_t*>(out) + size_t(r) * n;
  double* od = static_cast<double*>(out) + size_t(r) * n;
  mt_block_generate(e, n, [&](int64_t k, uint64_t raw) {
    if (kind == 0)
      o64[k] = raw;
    else if (kind == 1)
      od[k] = mt_uniform(raw);
    else
      od[k] = 1.0 - mt_uniform(raw);
  });
  mt_block_store(e, state + size_t(r) * kMtN, idx + r);
}

}  // namespace

int mt64_create(mg_ctx* ctx, int32_t streams, const uint64_t* host_seeds, mg_mt64** out) {
  if (!ctx || !out || !host_seeds || streams < 1) return fail(MG_EINVAL, "mg_mt64_create: bad args");
  mg_mt64* g = new mg_mt64();
  g->streams = streams;
  uint64_t* dseeds = nullptr;
  cudaError_t e = cudaMalloc(&g->state, sizeof(uint64_t) * kMtN * size_t(streams));
  if (e == cudaSuccess) e = cudaMalloc(&g->idx, sizeof(int) * size_t(streams));
  if (e == cudaSuccess) e = cudaMalloc(&dseeds, sizeof(uint64_t) * size_t(streams));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(dseeds, host_seeds, sizeof(uint64_t) * size_t(streams),
                        cudaMemcpyHostToDevice, ctx->stream);
  if (e != cudaSuccess) {
    cudaFree(dseeds);
    mt64_destroy(g);
    return cuda_fail(e, "mg_mt64_create");
  }
  mt_seed_kernel<<<(streams + 127) / 128, 128, 0, ctx->stream>>>(streams, dseeds, g->state, g->idx);
  ctx->launches++;
  e = cudaGetLastError();
  cudaStreamSynchronize(ctx->stream);
  cudaFree(dseeds);
  if (e != cudaSuccess) {
    mt64_destroy(g);
    return cuda_fail(e, "mt_seed_kernel");
  }
  *out = g;
  return MG_OK;
}

void mt64_destroy(mg_mt64* g) {
  if (!g) return;
  cudaFree(g->state);
  cudaFree(g->idx);
  delete g;
}

int mt64_draw(mg_ctx* ctx, mg_mt64* g, int64_t n, int32_t kind, void* out) {
  if (!ctx || !g || !out || n < 0 || kind < 0 || kind > 2)
    return fail(MG_EINVAL, "mg_mt64_draw: bad args");
  if (n == 0) return MG_OK;
  mt_draw_kernel<<<g->streams, kDrawThreads, 0, ctx->stream>>>(n, kind, g->state, g->idx, out);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

}  // namespace mg

extern "C" {

int mg_mt64_create(mg_ctx* ctx, int32_t streams, const uint64_t* host_seeds, mg_mt64** out) {
  return mg::mt64_create(ctx, streams, host_seeds, out);
}

int mg_mt64_destroy(mg_mt64* g) {
  mg::mt64_destroy(g);
  return MG_OK;
}

int mg_mt64_draw(mg_ctx* ctx, mg_mt64* g, int64_t n, int32_t kind, void* out) {
  return mg::mt64_draw(ctx, g, n, kind, out);
}

}  // extern "C"
