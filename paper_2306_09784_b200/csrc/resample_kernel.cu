// resample_kernel: polar image (Measure E) -> Cartesian grid "for comparability"
// (P:L365).  Bilinear interpolation of the complex values in (bearing, range) at each
// Cartesian pixel centre (in the x-y plane); pixels outside the polar coverage get 0.
#include <algorithm>

#include "sar_internal.h"

namespace sar {
namespace {

__global__ void polar_to_cart_kernel(const ResampleArgs a) {
  const long n = (long)a.nx * a.ny;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < n; idx += (long)gridDim.x * blockDim.x) {
    const int ix = (int)(idx % a.nx), iy = (int)(idx / a.nx);
    const double px = a.x0 + ix * a.dx - a.xc, py = a.y0 + iy * a.dy - a.yc;
    const double rr = sqrt(px * px + py * py);
    // bearing from +y toward +x relative to the sector centre, wrapped into [-pi, pi) (a sector
    // may cross +-pi and th0 may be given in any period; reading A19)
    const double half = 0.5 * (a.n_th - 1) * a.dth;
    double db = atan2(px, py) - (a.th0 + half);
    db -= 2.0 * kPi * floor((db + kPi) / (2.0 * kPi));
    double fi = (db + half) / a.dth, fj = (rr - a.r0) / a.dr;
    float2 v = make_float2(0.f, 0.f);
    // nodes on the sector boundary count as inside (1e-9 of an index of rounding slack)
    if (fi >= -1e-9 && fj >= -1e-9 && fi <= a.n_th - 1 + 1e-9 && fj <= a.n_r - 1 + 1e-9) {
      fi = fmin(fmax(fi, 0.0), (double)(a.n_th - 1));
      fj = fmin(fmax(fj, 0.0), (double)(a.n_r - 1));
      const int i0 = min((int)fi, a.n_th - 1), j0 = min((int)fj, a.n_r - 1);
      const int i1 = min(i0 + 1, a.n_th - 1), j1 = min(j0 + 1, a.n_r - 1);
      const float wi = (float)(fi - i0), wj = (float)(fj - j0);
      const float2 c00 = a.in[(size_t)j0 * a.n_th + i0], c01 = a.in[(size_t)j0 * a.n_th + i1];
      const float2 c10 = a.in[(size_t)j1 * a.n_th + i0], c11 = a.in[(size_t)j1 * a.n_th + i1];
      const float w00 = (1.f - wi) * (1.f - wj), w01 = wi * (1.f - wj), w10 = (1.f - wi) * wj, w11 = wi * wj;
      v.x = w00 * c00.x + w01 * c01.x + w10 * c10.x + w11 * c11.x;
      v.y = w00 * c00.y + w01 * c01.y + w10 * c10.y + w11 * c11.y;
    }
    a.out[idx] = v;
  }
}

}  // namespace

cudaError_t launch_resample(const ResampleArgs& a, cudaStream_t s) {
  const long n = (long)a.nx * a.ny;
  const int block = 256;
  const long grid = std::max(1L, std::min<long>((n + block - 1) / block, 148L * 32));
  polar_to_cart_kernel<<<(unsigned)grid, block, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sar
