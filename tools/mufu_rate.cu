// Microbenchmark: MUFU (XU pipe) and FFMA issue rates on sm_100a, results per SM per clock.
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void kern(float* out, int iters, float seed) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) {  // sin + cos of one argument (two MUFU)
        float s, c;
        __sincosf(a[i], &s, &c);
        a[i] = s + c;
      } else if (KIND == 1) {  // rsqrt
        float r;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a[i]));
        a[i] = r + 1.0f;
      } else if (KIND == 2) {  // sin only
        a[i] = __sinf(a[i]) + 1.5f;
      } else {  // FFMA only
        a[i] = fmaf(a[i], 0.999f, 0.001f);
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
  const char* names[] = {"sincos (2 MUFU/op)", "rsqrt", "sin", "ffma"};
  const int iters = 4096;
  for (int kind = 0; kind < 4; ++kind) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      const int blocks = sms * 8, threads = 256;
      if (kind == 0) kern<0><<<blocks, threads>>>(out, iters, 0.1f);
      if (kind == 1) kern<1><<<blocks, threads>>>(out, iters, 0.1f);
      if (kind == 2) kern<2><<<blocks, threads>>>(out, iters, 0.1f);
      if (kind == 3) kern<3><<<blocks, threads>>>(out, iters * 8, 0.1f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 8 * (kind == 3 ? 8 : 1);
      double per_sm_clk = ops / (ms * 1e-3) / sms / (clk * 1e3);
      if (rep) printf("%-20s %8.3f ms  %6.2f ops/clk/SM (at max clock %d MHz)\n", names[kind], ms, per_sm_clk, clk / 1000);
    }
  }
  return 0;
}
