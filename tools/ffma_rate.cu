// Microbenchmark: FFMA throughput on sm_100a with immediate vs. three register operands,
// and register-bank effects.  Reports lane-ops per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long rd;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&rd);
}

template <int KIND>
__global__ void __launch_bounds__(256) kern(float* out, int iters, float s0) {
  float a[8], b[8], c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = s0 + threadIdx.x * 1e-6f + i;
    b[i] = __shfl_sync(0xffffffffu, 0.9999f + 1e-7f * i, threadIdx.x & 31);
    c[i] = __shfl_sync(0xffffffffu, 1e-4f * i, threadIdx.x & 31);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) a[i] = fmaf(a[i], 0.9999f, 1e-4f);        // imm / const operands
      if (KIND == 1) a[i] = fmaf(a[i], b[i], c[i]);            // three distinct registers
      if (KIND == 2) a[i] = fmaf(a[i], b[0], c[0]);            // shared b, c (reuse-friendly)
      if (KIND == 3) a[i] = a[i] * b[i];                       // FMUL two registers
      if (KIND == 4) a[i] = a[i] + b[i];                       // FADD two registers
    }
    if (KIND == 5) {  // FFMA2, three distinct register pairs (2 FMA per lane per instruction)
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        float2 r = ffma2(make_float2(a[i], a[i + 1]), make_float2(b[i], b[i + 1]), make_float2(c[i], c[i + 1]));
        a[i] = r.x; a[i + 1] = r.y;
      }
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        float2 r = ffma2(make_float2(a[i], a[i + 1]), make_float2(b[i], b[i + 1]), make_float2(c[i], c[i + 1]));
        a[i] = r.x; a[i + 1] = r.y;
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
  const char* names[] = {"FFMA imm", "FFMA 3 distinct regs", "FFMA shared b,c regs", "FMUL 2 regs", "FADD 2 regs", "FFMA2 3 distinct pairs"};
  const int iters = 1 << 14, blocks = sms * 8, threads = 256;
  for (int kind = 0; kind < 6; ++kind) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (kind == 0) kern<0><<<blocks, threads>>>(out, iters, 0.1f);
      if (kind == 1) kern<1><<<blocks, threads>>>(out, iters, 0.1f);
      if (kind == 2) kern<2><<<blocks, threads>>>(out, iters, 0.1f);
      if (kind == 3) kern<3><<<blocks, threads>>>(out, iters, 0.1f);
      if (kind == 4) kern<4><<<blocks, threads>>>(out, iters, 0.1f);
      if (kind == 5) kern<5><<<blocks, threads>>>(out, iters, 0.1f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)blocks * threads * iters * 8;
      if (rep) printf("%-24s %8.3f ms  %7.2f lane-ops/clk/SM\n", names[kind], ms, ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
  }
  return 0;
}
