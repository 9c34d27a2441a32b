// Standalone HBM probe (nvcc -gencode arch=compute_100a,code=sm_100a -O3):
// how fast can ANY kernel stream the fused meta update's access pattern —
// 8 read and 6 written fp32 arrays of n = 2^28 — with no arithmetic?
// Prints GB/s (algorithmic bytes / kernel time, CUDA events, mean of 20
// back-to-back launches after 5 warm-up launches)
// for: a plain copy (1 read, 1 write), and 8-read/6-write register
// streaming with 16-byte loads/stores at several grid shapes.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_k(long n4, const float4* __restrict__ a, float4* __restrict__ b) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}

struct P {
  const float4* in[8];
  float4* out[6];
};

template <int U>
__global__ void mix_k(long n4, P p) {
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i0 = blockIdx.x * (long)blockDim.x + threadIdx.x; i0 < n4; i0 += stride * U) {
    float4 v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long i = i0 + u * stride;
      if (i < n4)
#pragma unroll
        for (int a = 0; a < 8; ++a) v[u][a] = __ldcs(p.in[a] + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long i = i0 + u * stride;
      if (i < n4)
#pragma unroll
        for (int a = 0; a < 6; ++a) {
          float4 x = v[u][a];
          x.x += v[u][6].x + v[u][7].x;
          __stcs(p.out[a] + i, x);
        }
    }
  }
}

int main() {
  const long n = 1L << 28, n4 = n / 4;
  float4* buf[14];
  for (int k = 0; k < 14; ++k) {
    cudaMalloc(&buf[k], n * 4);
    cudaMemset(buf[k], 0, n * 4);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // mean over 20 back-to-back launches after 5 warm-up launches (the
  // steady state bench.py reports), like the fused update's 20-step line
  auto timeit = [&](auto launch) {
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 20;
  };
  for (int bpsm : {4, 8, 16}) {
    const float ms = timeit([&] { copy_k<<<sms * bpsm, 256>>>(n4, buf[0], buf[1]); });
    printf("copy        grid %3d x 256: %.3f ms  %.0f GB/s\n", sms * bpsm, ms, 8.0 * n / ms / 1e6);
  }
  P p;
  for (int a = 0; a < 8; ++a) p.in[a] = buf[a];
  for (int a = 0; a < 6; ++a) p.out[a] = buf[8 + a];
  for (int th : {128, 256, 512})
    for (int bpsm : {2, 4, 8}) {
      float ms = timeit([&] { mix_k<1><<<sms * bpsm, th>>>(n4, p); });
      printf("mix8r6w U1 grid %3d x %3d: %.3f ms  %.0f GB/s\n", sms * bpsm, th, ms, 56.0 * n / ms / 1e6);
      ms = timeit([&] { mix_k<2><<<sms * bpsm, th>>>(n4, p); });
      printf("mix8r6w U2 grid %3d x %3d: %.3f ms  %.0f GB/s\n", sms * bpsm, th, ms, 56.0 * n / ms / 1e6);
    }
  return 0;
}
