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

// Chirp-split sum, one CTA per tile of the launch: pixel (x, y) of the tile (holding chunk 0's
// store, or its accumulation) gets + ws[0] + ws[1] + ... in chunk order.  Rows of a
// tile are 32 contiguous pixels (256 B), so each warp reads and writes whole rows.
__global__ void __launch_bounds__(256) split_sum_kernel(const SplitSumArgs a) {
  const int tile = a.tile0 + blockIdx.x;
  const int i0 = (tile % a.tiles_x) * kTileX, J0 = (tile / a.tiles_x) * a.tile_y;
  const int x = i0 + (threadIdx.x & 31);
  if (x >= a.nx) return;
  for (int yl = threadIdx.x >> 5; yl < a.tile_y; yl += blockDim.x >> 5) {
    const int y = J0 + yl - a.row0;
    if (y < 0 || y >= a.nrow) continue;
    const size_t o = (size_t)y * a.nx + x;
    float2 s = a.img[o];
    for (int c = 0; c < a.planes; ++c) {
      const float2 v = __ldcs(a.ws + (size_t)c * a.plane + o);
      s.x += v.x;
      s.y += v.y;
    }
    a.img[o] = s;
  }
}

// One CTA per tile, one warp per 32-pixel tile row: every finished pixel is read once from the
// local image and stored to each peer image (coalesced 256-B rows, P2P over NVLink).
__global__ void __launch_bounds__(256) publish_kernel(const PublishArgs a) {
  const int tile = a.tile0 + blockIdx.x;
  const int i0 = (tile % a.tiles_x) * kTileX, J0 = (tile / a.tiles_x) * a.tile_y;
  const int x = i0 + (threadIdx.x & 31);
  if (x >= a.nx) return;
  for (int yl = threadIdx.x >> 5; yl < a.tile_y; yl += blockDim.x >> 5) {
    const int y = J0 + yl;
    if (y >= a.ny) break;
    const size_t o = (size_t)y * a.nx + x;
    const float2 v = __ldcs(a.src + o);
    for (int d = 0; d < a.n_dst; ++d) a.dst[d][o] = v;
  }
}

}  // namespace

cudaError_t launch_publish(const PublishArgs& a, cudaStream_t s) {
  if (a.ntile <= 0 || a.n_dst <= 0) return cudaSuccess;
  publish_kernel<<<(unsigned)a.ntile, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_split_sum(const SplitSumArgs& a, cudaStream_t s) {
  if (a.ntile <= 0) return cudaSuccess;
  split_sum_kernel<<<(unsigned)a.ntile, 256, 0, s>>>(a);
  return cudaGetLastError();
}

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
