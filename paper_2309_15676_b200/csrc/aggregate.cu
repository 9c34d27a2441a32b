// F2: across-replicate aggregation on the device.
//
// The reference reduces the per-replicate series of run_experiment on the
// host, iteration by iteration (harness.cpp:274-302): for every (series,
// iteration) column it collects the values of the replicates still active
// (iterations_run > i) in replicate order and takes mean_of, variance_of and
// the 0.5/0.25/0.75 linear-interpolation quantiles (stats.hpp:44-68).
//
// Here one CTA owns one column.  The values are staged in shared memory
// twice: in replicate order (the sums of mean_of / variance_of are
// sequential in the reference, so one thread walks them in that order and
// the results are bit-identical) and compacted for a block-wide bitonic sort
// (order of equal keys is irrelevant to the quantiles).  NaN sorts after
// every number — numpy's convention; std::sort's order with NaN present is
// unspecified.  Only the [S][5][T] statistics leave the device, instead of
// the [S][R][T] series.
#include <math.h>

#include "mg_common.cuh"

namespace mg {
namespace {

constexpr int kAggThreads = 256;
constexpr int kAggMaxReplicates = 8192;

__device__ __forceinline__ bool agg_less(double a, double b) {
  return a < b || (!isnan(a) && isnan(b));
}

__device__ __forceinline__ double agg_quantile(const double* s, int m, double p) {
  // stats.hpp:45-53 on the sorted sample
  const double pos = p * double(m - 1);
  const int lo = int(pos);
  if (lo + 1 >= m) return s[m - 1];
  const double frac = pos - double(lo);
  return s[lo] * (1.0 - frac) + s[lo + 1] * frac;
}

// series [S][R][T], runs[r * runs_stride] = iterations_run of replicate r,
// stats [S][5][T] = mean, variance, median, q25, q75; active[T].
__global__ void __launch_bounds__(kAggThreads)
    aggregate_kernel(int S, int R, int T, const double* __restrict__ series,
                     const int32_t* __restrict__ runs, int runs_stride,
                     double* __restrict__ stats, int32_t* __restrict__ active) {
  extern __shared__ double agg_sm[];
  double* ord = agg_sm;            // [R]  replicate order (NaN-free flags below)
  double* srt = agg_sm + R;        // [P]  compacted, sorted
  __shared__ int cnt;
  const int col = blockIdx.x;
  const int s = col / T, i = col - s * T;
  const double* x = series + size_t(s) * R * T + i;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < R; r += kAggThreads) {
    const bool act = runs[size_t(r) * runs_stride] > i;
    const double v = act ? x[size_t(r) * T] : 0.0;
    ord[r] = v;
    if (act) srt[atomicAdd(&cnt, 1)] = v;
  }
  __syncthreads();
  const int m = cnt;
  int P = 1;
  while (P < m) P <<= 1;
  for (int k = m + threadIdx.x; k < P; k += kAggThreads) srt[k] = __longlong_as_double(0x7ff8000000000000LL);
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (P >> 1); t += kAggThreads) {
        const int a = 2 * t - (t & (stride - 1));
        const int b = a + stride;
        const bool up = (a & size) == 0;
        const double va = srt[a], vb = srt[b];
        if (agg_less(vb, va) == up) {
          srt[a] = vb;
          srt[b] = va;
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    double mean = __longlong_as_double(0x7ff8000000000000LL), var = 0.0;
    double med = mean, q25 = mean, q75 = mean;
    if (m > 0) {
      // mean_of / variance_of: sequential sums in replicate order
      double acc = 0.0;
      for (int r = 0; r < R; ++r)
        if (runs[size_t(r) * runs_stride] > i) acc += ord[r];
      mean = acc / double(m);
      if (m >= 2) {
        double sq = 0.0;
        for (int r = 0; r < R; ++r)
          if (runs[size_t(r) * runs_stride] > i) sq += (ord[r] - mean) * (ord[r] - mean);
        var = sq / double(m - 1);
      }
      med = agg_quantile(srt, m, 0.5);
      q25 = agg_quantile(srt, m, 0.25);
      q75 = agg_quantile(srt, m, 0.75);
    }
    double* o = stats + size_t(s) * 5 * T + i;
    o[0] = mean;
    o[size_t(T)] = var;
    o[2 * size_t(T)] = med;
    o[3 * size_t(T)] = q25;
    o[4 * size_t(T)] = q75;
    if (s == 0 && active) active[i] = m;
  }
}

}  // namespace

size_t aggregate_smem_bytes(int R) {
  int P = 1;
  while (P < R) P <<= 1;
  return sizeof(double) * (size_t(R) + size_t(P));
}

int launch_aggregate(mg_ctx* ctx, int S, int R, int T, const double* series, const int32_t* runs,
                     int runs_stride, double* stats, int32_t* active) {
  if (S < 1 || R < 1 || T < 1) return fail(MG_EINVAL, "aggregate: bad sizes");
  if (R > kAggMaxReplicates)
    return fail(MG_EUNSUPPORTED, "aggregate: more than 8192 replicates per column");
  if (int64_t(S) * T > 0x7fffffffLL) return fail(MG_EINVAL, "aggregate: too many columns");
  const size_t smem = aggregate_smem_bytes(R);
  MG_CUDA_TRY(cudaFuncSetAttribute(aggregate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
  aggregate_kernel<<<S * T, kAggThreads, smem, ctx->stream>>>(S, R, T, series, runs, runs_stride,
                                                              stats, active);
  MG_LAUNCH_CHECK(ctx);
  return MG_OK;
}

}  // namespace mg

extern "C" int mg_aggregate_series(mg_ctx* ctx, int32_t S, int32_t R, int32_t T,
                                   const double* series, const int32_t* iterations_run,
                                   double* stats, int32_t* active) {
  if (!ctx || !series || !iterations_run || !stats)
    return mg::fail(MG_EINVAL, "mg_aggregate_series: null argument");
  return mg::launch_aggregate(ctx, S, R, T, series, iterations_run, 1, stats, active);
}
