// Batched device std::mt19937_64 engines (row A1, rng.hpp:18-37).
#include <vector>

#include "mg_common.cuh"
#include "mt64.cuh"
#include "mt64_state.h"
#include "mt64_jump.h"

#include <map>
#include <mutex>

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

// GF(2) jump-ahead of every stream (Haramoto et al. 2008, see
// mt64_jump.cu): R = g(A) W by Horner's rule in base 16, one warp per
// stream.  W is the state window (x_t .. x_{t+311}) = the stored buffer of a
// stream sitting at a block boundary (idx == 312).  Streams with mask[r]==0
// (when a mask is given) are left untouched.
constexpr int kJumpThreads = 32;
constexpr size_t kJumpSmem = sizeof(uint64_t) * (16 * kMtN + kMtN + kMtN + 3 + kMtN);

__global__ void __launch_bounds__(kJumpThreads)
    mt_jump_kernel(int streams, uint64_t* __restrict__ state, const int* __restrict__ idx,
                   const uint64_t* __restrict__ g, int deg, const uint8_t* __restrict__ mask,
                   int* __restrict__ bad) {
  extern __shared__ uint64_t sm[];
  uint64_t* T = sm;                  // [16][312]: T[m] = sum_{j in m} A^j W
  uint64_t* R = sm + 16 * kMtN;      // circular window, start s
  uint64_t* E = R + kMtN;            // W followed by 3 new words
  uint64_t* G = E + kMtN + 3;        // the jump polynomial
  const int r = blockIdx.x;
  const int lane = threadIdx.x;
  if (mask && !mask[r]) return;
  if (idx[r] != kMtN) {
    if (lane == 0) *bad = 1;
    return;
  }
  uint64_t* st = state + size_t(r) * kMtN;
  for (int c = lane; c < kMtN; c += kJumpThreads) {
    E[c] = st[c];
    R[c] = 0;
    G[c] = g[c];
  }
  __syncwarp();
  if (lane < 3) {
    // y_i = E[i+156] ^ mag(E[i], E[i+1]) for i = 0..2 (all inputs are in W)
    E[kMtN + lane] = E[lane + kMtM] ^ mt_mag(E[lane], E[lane + 1]);
  }
  __syncwarp();
  for (int c = lane; c < kMtN; c += kJumpThreads) {
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      uint64_t v = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (m & (1 << j)) v ^= E[j + c];
      T[m * kMtN + c] = v;
    }
  }
  __syncwarp();
  int s = 0;  // R canonical word c lives at R[(s + c) mod 312]
  constexpr int kPer = (kMtN + kJumpThreads - 1) / kJumpThreads;  // 10 words per lane
  const int top = deg < 0 ? -1 : deg / 4;
  int digit_next = top >= 0 ? int((G[(4 * top) >> 6] >> ((4 * top) & 63)) & 0xFu) : 0;
  for (int k = top; k >= 0; --k) {
    const int digit = digit_next;
    if (k > 0) digit_next = int((G[(4 * (k - 1)) >> 6] >> ((4 * (k - 1)) & 63)) & 0xFu);
    // R = A^4 R: four new words from the current window (independent), then
    // they replace the 4 words shifted out
    uint64_t y = 0;
    if (lane < 4) {
      int i0 = s + lane, i1 = i0 + 1, i2 = i0 + kMtM;
      i0 -= i0 >= kMtN ? kMtN : 0;
      i1 -= i1 >= kMtN ? kMtN : 0;
      i2 -= i2 >= kMtN ? kMtN : 0;
      y = R[i2] ^ mt_mag(R[i0], R[i1]);
    }
    __syncwarp();
    if (lane < 4) {
      int w = s + lane;
      R[w - (w >= kMtN ? kMtN : 0)] = y;
    }
    s += 4;
    s -= s >= kMtN ? kMtN : 0;
    __syncwarp();
    if (digit) {
      // R ^= T[digit]: all loads first (ILP), then the stores
      const uint64_t* t = T + digit * kMtN;
      uint64_t v[kPer];
      int at[kPer];
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int c = lane + i * kJumpThreads;
        int w = s + c;
        w -= w >= kMtN ? kMtN : 0;
        at[i] = w;
        v[i] = c < kMtN ? (R[w < kMtN ? w : 0] ^ t[c < kMtN ? c : 0]) : 0;
      }
#pragma unroll
      for (int i = 0; i < kPer; ++i)
        if (lane + i * kJumpThreads < kMtN) R[at[i]] = v[i];
    }
    __syncwarp();
  }
  for (int c = lane; c < kMtN; c += kJumpThreads) st[c] = R[(s + c) % kMtN];
}

}  // namespace

// Host cache of jump polynomials (computing one costs ~0.1 s).
struct JumpPoly {
  uint64_t* dev = nullptr;
  int deg = -1;
};

static int get_jump_poly(uint64_t distance, JumpPoly* out) {
  static std::mutex mu;
  static std::map<uint64_t, JumpPoly> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(distance);
  if (it != cache.end()) {
    *out = it->second;
    return MG_OK;
  }
  std::vector<uint64_t> w(kMtJumpWords);
  int deg = -1;
  if (!mt64_jump_polynomial(distance, w.data(), &deg))
    return fail(MG_ELOGIC, "mt19937_64 characteristic polynomial: unexpected degree");
  JumpPoly jp;
  jp.deg = deg;
  MG_CUDA_TRY(cudaMalloc(&jp.dev, sizeof(uint64_t) * kMtJumpWords));
  MG_CUDA_TRY(cudaMemcpy(jp.dev, w.data(), sizeof(uint64_t) * kMtJumpWords,
                         cudaMemcpyHostToDevice));
  // a pageable cudaMemcpy may return before its DMA lands; the jump kernel
  // runs on a (possibly non-blocking) context stream, so fence the device
  MG_CUDA_TRY(cudaDeviceSynchronize());
  cache[distance] = jp;
  *out = jp;
  return MG_OK;
}

int mt64_jump(mg_ctx* ctx, mg_mt64* g, uint64_t distance, const uint8_t* dev_mask) {
  if (!ctx || !g) return fail(MG_EINVAL, "mg_mt64_jump: null argument");
  if (distance == 0) return MG_OK;
  JumpPoly jp;
  int st = get_jump_poly(distance, &jp);
  if (st) return st;
  static bool attr_set = false;
  if (!attr_set) {
    MG_CUDA_TRY(cudaFuncSetAttribute(mt_jump_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kJumpSmem)));
    attr_set = true;
  }
  // All streams of a batch draw the same counts, so their block position is
  // tracked on the host (no device round trip); the kernel re-checks.
  if (g->host_idx != kMtN)
    return fail(MG_EINVAL, "mg_mt64_jump: the streams are not at a 312-draw block boundary "
                           "(draw multiples of 312 between jumps)");
  mt_jump_kernel<<<g->streams, kJumpThreads, kJumpSmem, ctx->stream>>>(
      g->streams, g->state, g->idx, jp.dev, jp.deg, dev_mask, ctx->flag);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

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
  g->host_idx = int((int64_t(g->host_idx) + n - 1) % kMtN) + 1;  // position after n draws
  mt_draw_kernel<<<g->streams, kDrawThreads, 0, ctx->stream>>>(n, kind, g->state, g->idx, out);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

}  // namespace mg

extern "C" {

int mg_mt64_jump(mg_ctx* ctx, mg_mt64* g, uint64_t distance) {
  return mg::mt64_jump(ctx, g, distance, nullptr);
}

// `segments` engines on ONE stream: engine c starts c*segment_len draws
// into the stream seeded with engine_seed (binary decomposition of c into
// jumps by 2^i * segment_len, masked per engine).
int mg_mt64_split(mg_ctx* ctx, uint64_t engine_seed, int32_t segments, uint64_t segment_len,
                  mg_mt64** out) {
  using namespace mg;
  if (!ctx || !out || segments < 1) return fail(MG_EINVAL, "mg_mt64_split: bad arguments");
  std::vector<uint64_t> seeds(size_t(segments), engine_seed);
  mg_mt64* g = nullptr;
  int st = mt64_create(ctx, segments, seeds.data(), &g);
  if (st) return st;
  uint8_t* dmask = nullptr;
  MG_CUDA_TRY(cudaMalloc(&dmask, size_t(segments)));
  std::vector<uint8_t> mask(static_cast<size_t>(segments));
  for (int bit = 0; bit < 31 && (int64_t(1) << bit) < segments; ++bit) {
    for (int c = 0; c < segments; ++c) mask[size_t(c)] = uint8_t((c >> bit) & 1);
    // ordered on the context's stream: the previous jump may still be
    // reading the mask (the stream need not synchronise with the legacy one)
    cudaMemcpyAsync(dmask, mask.data(), size_t(segments), cudaMemcpyHostToDevice, ctx->stream);
    st = mt64_jump(ctx, g, segment_len << bit, dmask);
    if (st) break;
  }
  cudaStreamSynchronize(ctx->stream);
  cudaFree(dmask);
  if (st) {
    mt64_destroy(g);
    return st;
  }
  *out = g;
  return MG_OK;
}

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

// The engine state in libstdc++'s std::mt19937_64 layout (_M_x[312], _M_p;
// random.h:1620-1627, serialised by its operator<< / operator>>), so a host
// engine can hand its position to the device and take it back.
int mg_mt64_set_state(mg_ctx* ctx, mg_mt64* g, int32_t stream, const uint64_t* words,
                      int32_t idx) {
  using namespace mg;
  if (!ctx || !g || !words) return fail(MG_EINVAL, "mg_mt64_set_state: null argument");
  if (stream < 0 || stream >= g->streams) return fail(MG_EINVAL, "mg_mt64_set_state: bad stream");
  if (idx < 0 || idx > kMtN) return fail(MG_EINVAL, "mg_mt64_set_state: index must lie in [0, 312]");
  MG_CUDA_TRY(cudaMemcpyAsync(g->state + size_t(stream) * kMtN, words, sizeof(uint64_t) * kMtN,
                              cudaMemcpyHostToDevice, ctx->stream));
  MG_CUDA_TRY(cudaMemcpyAsync(g->idx + stream, &idx, sizeof(int), cudaMemcpyHostToDevice,
                              ctx->stream));
  MG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  g->host_idx = idx;
  return MG_OK;
}

int mg_mt64_get_state(mg_ctx* ctx, mg_mt64* g, int32_t stream, uint64_t* words, int32_t* idx) {
  using namespace mg;
  if (!ctx || !g || !words || !idx) return fail(MG_EINVAL, "mg_mt64_get_state: null argument");
  if (stream < 0 || stream >= g->streams) return fail(MG_EINVAL, "mg_mt64_get_state: bad stream");
  int i = 0;
  MG_CUDA_TRY(cudaMemcpyAsync(words, g->state + size_t(stream) * kMtN, sizeof(uint64_t) * kMtN,
                              cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA_TRY(cudaMemcpyAsync(&i, g->idx + stream, sizeof(int), cudaMemcpyDeviceToHost,
                              ctx->stream));
  MG_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  *idx = i;
  return MG_OK;
}

}  // extern "C"
