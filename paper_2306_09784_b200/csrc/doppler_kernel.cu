// doppler_kernel: per-pixel Doppler index shift f_doppler(p) of Measure D,
// the input of Alg. 2 L8.  One thread per pixel, fp64 geometry, float32 output.
#include <algorithm>

#include "sar_internal.h"

namespace sar {
namespace {

__global__ void doppler_kernel(const DopArgs a) {
  const long n = (long)a.nx * a.ny;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const int ix = (int)(i % a.nx), iy = (int)(i / a.nx);
    double px, py;
    if (a.polar) {   // Measure E grid: (xc + r sin th, yc + r cos th), image [n_r][n_th]
      const double rr = a.r0 + iy * a.dr, th = a.th0 + ix * a.dth;
      px = a.x0 + rr * sin(th);
      py = a.y0 + rr * cos(th);
    } else {
      px = a.x0 + ix * a.dx;
      py = a.y0 + iy * a.dy;
    }
    const double dx = px - a.q[0];
    const double dy = py - a.q[1];
    const double dz = a.z0 - a.q[2];
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    const double vr = r > 0.0 ? a.legs * (dx * a.v[0] + dy * a.v[1] + dz * a.v[2]) / r : 0.0;
    a.out[i] = (float)(vr * a.bins_per_mps);
  }
}

}  // namespace

cudaError_t launch_doppler(const DopArgs& a, cudaStream_t s) {
  const long n = (long)a.nx * a.ny;
  const int block = 256;
  const long grid = std::min<long>((n + block - 1) / block, 148L * 32);
  doppler_kernel<<<(unsigned)grid, block, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sar
