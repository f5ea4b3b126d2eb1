// Microbenchmark: do MUFU (XU) and LDS.128 share one MIO throughput limit on sm_100a?
// Each "update" = NM MUFU + NL LDS.128 (broadcast-light gather) + NF FFMA, 4 independent
// chains per thread, 8 warps x 4 CTAs per SM.  Prints SM clocks per warp-update.
#include <cstdio>
#include <cuda_runtime.h>

template <int NM, int NL, int NF>
__global__ void __launch_bounds__(256) kern(float* out, int iters) {
  __shared__ float4 tab[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) tab[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float a[4], acc[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) { a[p] = 0.001f * threadIdx.x + p; acc[p] = 0.f; }
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      float x = a[p];
#pragma unroll
      for (int f = 0; f < NF; ++f) x = fmaf(x, 0.9999f, 1e-4f);
      float m = 0.f;
#pragma unroll
      for (int k = 0; k < NM; ++k) m += __sinf(x + k);
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const int idx = ((lane >> 3) + (__float_as_int(x) & 3) + 8 * p + 16 * l) & 511;
        const float4 v = tab[idx];
        m += v.x + v.w;
      }
      acc[p] += m;
      a[p] = x;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3];
}

template <int NM, int NL, int NF>
void run(const char* name, float* out, int sms, int clk_khz) {
  const int iters = 2048, blocks = sms * 4, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<NM, NL, NF><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_updates_per_sm = (double)blocks * threads / 32 * iters * 4 / sms;
    const double clk = ms * 1e-3 * clk_khz * 1e3;
    if (rep) printf("%-34s %7.3f ms  %6.2f SM-clk per warp-update\n", name, ms, clk / warp_updates_per_sm);
  }
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 4 * 256);
  run<3, 0, 20>("3 MUFU + 20 FFMA", out, sms, clk);
  run<3, 1, 20>("3 MUFU + 1 LDS.128 + 20 FFMA", out, sms, clk);
  run<0, 1, 20>("1 LDS.128 + 20 FFMA", out, sms, clk);
  run<2, 1, 20>("2 MUFU + 1 LDS.128 + 20 FFMA", out, sms, clk);
  run<3, 2, 20>("3 MUFU + 2 LDS.128 + 20 FFMA", out, sms, clk);
  run<3, 0, 0>("3 MUFU", out, sms, clk);
  run<0, 4, 0>("4 LDS.128", out, sms, clk);
  run<0, 0, 24>("24 FFMA", out, sms, clk);
  return 0;
}
