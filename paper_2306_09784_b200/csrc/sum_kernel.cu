// sum_kernel: frame = sum of the per-hop partial images of a world-fixed grid (incremental
// streaming, NEXT-2).  HBM-bound: reads n_partials x 8 B and writes 8 B per pixel, float4
// (two complex pixels) per thread, grid-stride over a multiple of the SM count.
#include <algorithm>

#include "sar_internal.h"

namespace sar {
namespace {

__global__ void sum_kernel(float2* __restrict__ out, const float2* __restrict__ in, int n, long stride, long count) {
  const long pairs = count >> 1;
  const float4* in4 = reinterpret_cast<const float4*>(in);
  float4* out4 = reinterpret_cast<float4*>(out);
  const bool vec = ((stride & 1) == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  const long step = (long)gridDim.x * blockDim.x;
  if (vec) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < pairs; i += step) {
      float4 s = __ldg(in4 + i);
      for (int k = 1; k < n; ++k) {
        const float4 v = __ldg(in4 + k * (stride >> 1) + i);
        s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
      }
      out4[i] = s;
    }
    for (long i = 2 * pairs + blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += step) {
      float2 s = in[i];
      for (int k = 1; k < n; ++k) { const float2 v = in[k * stride + i]; s.x += v.x; s.y += v.y; }
      out[i] = s;
    }
  } else {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += step) {
      float2 s = in[i];
      for (int k = 1; k < n; ++k) { const float2 v = in[k * stride + i]; s.x += v.x; s.y += v.y; }
      out[i] = s;
    }
  }
}

}  // namespace

cudaError_t launch_sum(float2* out, const float2* in, int n, long stride, long count, cudaStream_t s) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int block = 256;
  const long want = (count / 2 + block - 1) / block;
  const long grid = std::max(1L, std::min(want, (long)sms * 8));
  sum_kernel<<<(unsigned)grid, block, 0, s>>>(out, in, n, stride, count);
  return cudaGetLastError();
}

}  // namespace sar
