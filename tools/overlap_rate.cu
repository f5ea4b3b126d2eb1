// Microbenchmark: do MUFU (XU pipe) and FFMA (FMA pipe) instructions overlap on sm_100a?
// 8 independent chains per thread; per iteration each chain runs NM MUFU.RSQ and NF FFMA
// (immediate form, or three-register form when REG).  Time per warp-instruction mix is
// compared with the MUFU-only and FFMA-only runs: overlap -> max, shared issue -> sum.
#include <cstdio>
#include <cuda_runtime.h>

template <int NM, int NF, bool REG, bool PAIR>
__global__ void __launch_bounds__(256) kern(float* out, int iters, float b0, float c0) {
  float x[8], b[8], c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = 1.0f + 1e-3f * (threadIdx.x & 31) + 0.01f * i;
    b[i] = __shfl_sync(0xffffffffu, b0 + 1e-7f * i, threadIdx.x & 31);
    c[i] = __shfl_sync(0xffffffffu, c0 + 1e-7f * i, threadIdx.x & 31);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float v = x[i];
#pragma unroll
      for (int m = 0; m < NM; ++m) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(v));
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        if (PAIR) {
          // packed pair (FFMA2) with three distinct register pairs, counted as 2 FFMA
          unsigned long long vv, bb, cc;
          asm("mov.b64 %0, {%1, %2};" : "=l"(vv) : "f"(v), "f"(x[(i + 1) & 7]));
          asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b[i]), "f"(b[(i + 3) & 7]));
          asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "f"(c[i]), "f"(c[(i + 5) & 7]));
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(vv) : "l"(bb), "l"(cc));
          float lo, hi;
          asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(vv));
          v = lo + 0.f * hi;
          ++f;
        } else if (REG) {
          asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v) : "f"(b[i]), "f"(c[i]));
        } else {
          asm volatile("fma.rn.f32 %0, %0, 0f3F7FF972, 0f38D1B717;" : "+f"(v));
        }
      }
      x[i] = v;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NM, int NF, bool REG, bool PAIR = false>
void run(float* out, int sms, int clk_khz) {
  const int iters = 1024, blocks = sms * 8, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<NM, NF, REG, PAIR><<<blocks, threads>>>(out, iters, 0.9999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // SMSP cycles per warp per chain-iteration
    const double warp_iters_per_smsp = (double)blocks * threads / 32 * iters * 8 / (sms * 4);
    const double clk = ms * 1e-3 * clk_khz * 1e3;
    if (rep)
      printf("NM=%d NF=%2d %-5s %7.3f ms  %6.2f SMSP-clk per chain-iter (MUFU alone %d, FFMA alone %s%d)\n", NM, NF,
             PAIR ? "pair" : REG ? "reg" : "imm", ms, clk / warp_iters_per_smsp, 8 * NM, REG || PAIR ? "2x" : "", NF);
  }
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
  run<1, 0, false>(out, sms, clk);
  run<0, 8, false>(out, sms, clk);
  run<1, 4, false>(out, sms, clk);
  run<1, 8, false>(out, sms, clk);
  run<1, 12, false>(out, sms, clk);
  run<0, 8, true>(out, sms, clk);
  run<1, 4, true>(out, sms, clk);
  run<1, 8, true>(out, sms, clk);
  run<0, 8, false, true>(out, sms, clk);
  run<1, 8, false, true>(out, sms, clk);
  run<2, 8, false>(out, sms, clk);
  run<2, 16, false>(out, sms, clk);
  return 0;
}
