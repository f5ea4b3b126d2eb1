// pair_kernel: profiles -> pair-format rows for the BP producer's bulk copies.
// Entry i of a row holds, for the lower crop bin k = k0 + i - pad (k0 > 0: a row shard's
// own crop),
//   {mid = (X[k] + X[k+1]) / 2, diff = X[k+1] - X[k]} * exp(j 2 pi beta (k_lo + k + 1/2))
// with X = 0 outside the crop (A8): the same values the BP producer otherwise builds per
// (tile, chirp) window, built once per chirp row instead.  HBM-bound: 8 n_bins B read,
// 16 (n_bins + 2 pad) B written per row.
#include <algorithm>

#include "sar_internal.h"

namespace sar {
namespace {

__global__ void pair_kernel(const PairArgs a) {
  const long n = (long)a.rows * a.stride;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < n; idx += (long)gridDim.x * blockDim.x) {
    const long row = idx / a.stride;
    const int i = (int)(idx - row * a.stride);
    const int k = a.k0 + i - a.pad;
    const float2* x = a.prof + (size_t)(a.row0 + row) * a.n_bins;
    const float2 x0 = (k >= 0 && k < a.n_bins) ? __ldg(x + k) : make_float2(0.f, 0.f);
    const float2 x1 = (k + 1 >= 0 && k + 1 < a.n_bins) ? __ldg(x + k + 1) : make_float2(0.f, 0.f);
    const float2 q = __ldg(a.binphase + min(max(k, -1), a.n_bins - 1) + 1);
    const float mr = 0.5f * (x0.x + x1.x), mi = 0.5f * (x0.y + x1.y);
    const float dr = x1.x - x0.x, di = x1.y - x0.y;
    a.out[(size_t)(a.row0 + row) * a.stride + i] =
        make_float4(mr * q.x - mi * q.y, mr * q.y + mi * q.x, dr * q.x - di * q.y, dr * q.y + di * q.x);
  }
}

}  // namespace

cudaError_t launch_pairs(const PairArgs& a, cudaStream_t s) {
  const long n = (long)a.rows * a.stride;
  if (n == 0) return cudaSuccess;
  const int block = 256;
  const long grid = std::max(1L, std::min<long>((n + block - 1) / block, 148L * 32));
  pair_kernel<<<(unsigned)grid, block, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sar
