// rc_kernel: batched windowed, zero-padded, cropped real-to-complex range FFT (step H1).
//
//   X_{m,n}[k] = (2 w_sar[m] / sum w) sum_{t<Ns} w[t] x[t] exp(-j 2 pi k (t - t_c) / N)
//   for k in the plan's crop [k_lo, k_lo + n_bins)           (A4-A8)
//
// One CTA transforms TWO real rows at once (z = x_a + j x_b, the classic two-for-one real
// FFT), so one N-point complex FFT in shared memory serves two profiles.  The FFT is an
// in-place radix-4 decimation-in-frequency (one radix-2 pass first when log2 N is odd)
// with a float32 twiddle table built in double on the host; the output stays in
// digit-reversed order and the epilogue gathers only the cropped bins, separates the two
// real spectra, applies the centring ramp exp(+j 2 pi k t_c / N) and the scale, and
// stores coalesced complex64 rows.  HBM traffic per row: 4 Ns bytes read, 8 n_bins written.
#include <atomic>

#include "sar_internal.h"

namespace sar {
namespace {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// Reverse the log2n-bit index in base 4 (with a leading base-2 digit when log2n is odd).
__device__ __forceinline__ int digit_reverse(int k, int log2n) {
  // DIF with radix-2 first pass (if odd) then radix-4 passes produces output at
  // position p for frequency k where p is k with its mixed-radix digits reversed.
  // Mixed radix from the most significant end: [2 (if odd)], 4, 4, ..., 4.
  // Frequency k = d0 + r0 * (d1 + r1 * (...)) with the first-pass radix r0 as the
  // least-significant digit of k.
  int p = 0;
  int rem = log2n;
  if (log2n & 1) {            // first pass radix 2: its digit is k's LSB, becomes p's MSB
    p = (k & 1) << (log2n - 1);
    k >>= 1;
    rem -= 1;
  }
  // remaining radix-4 digits: k's next-least-significant digit goes to p's next-most position
  int shift = rem - 2;
  while (rem > 0) {
    p |= (k & 3) << shift;
    k >>= 2;
    shift -= 2;
    rem -= 2;
  }
  return p;
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) rc_kernel(const RcArgs a) {
  extern __shared__ float2 z[];  // [nfft]
  const int N = a.nfft;
  const int ra = a.row0 + 2 * blockIdx.x;          // first row of the pair
  const bool has_b = 2 * blockIdx.x + 1 < a.nrows;
  const float* xa = a.raw + (size_t)ra * a.ns;
  const float* xb = xa + a.ns;

  // load, window, zero-pad: z[t] = w[t] (x_a[t] + j x_b[t])
  for (int t = threadIdx.x; t < N; t += BLOCK) {
    float2 v = make_float2(0.f, 0.f);
    if (t < a.ns) {
      const float w = __ldg(a.window + t);
      v.x = w * __ldg(xa + t);
      v.y = has_b ? w * __ldg(xb + t) : 0.f;
    }
    z[t] = v;
  }
  __syncthreads();

  int len = N;  // current sub-transform length
  if (a.log2n & 1) {
    // radix-2 DIF pass over the whole array: pairs (i, i + N/2), twiddle W_N^i
    const int h = N >> 1;
    for (int i = threadIdx.x; i < h; i += BLOCK) {
      const float2 u = z[i], v = z[i + h];
      z[i] = make_float2(u.x + v.x, u.y + v.y);
      z[i + h] = cmul(make_float2(u.x - v.x, u.y - v.y), __ldg(a.twiddle + i));
    }
    len = h;
    __syncthreads();
  }
  // radix-4 DIF passes: sub-transforms of length len, quarter q = len/4
  int lq = a.log2n - (a.log2n & 1) - 2;            // log2 of the quarter length
  while (len >= 4) {
    const int q = len >> 2;
    const int stride = N / len;                    // twiddle index scale: W_len^j = W_N^(j*stride)
    const int nbf = N >> 2;                         // radix-4 butterflies per pass
    for (int b = threadIdx.x; b < nbf; b += BLOCK) {
      const int grp = b >> lq, j = b & (q - 1);
      const int i0 = (grp << (lq + 2)) + j;
      const float2 x0 = z[i0], x1 = z[i0 + q], x2 = z[i0 + 2 * q], x3 = z[i0 + 3 * q];
      const float2 s02 = make_float2(x0.x + x2.x, x0.y + x2.y);
      const float2 d02 = make_float2(x0.x - x2.x, x0.y - x2.y);
      const float2 s13 = make_float2(x1.x + x3.x, x1.y + x3.y);
      const float2 d13 = make_float2(x1.x - x3.x, x1.y - x3.y);
      // y0 = s02 + s13; y2 = s02 - s13; y1 = d02 - j d13; y3 = d02 + j d13
      const float2 y0 = make_float2(s02.x + s13.x, s02.y + s13.y);
      const float2 y2 = make_float2(s02.x - s13.x, s02.y - s13.y);
      const float2 y1 = make_float2(d02.x + d13.y, d02.y - d13.x);
      const float2 y3 = make_float2(d02.x - d13.y, d02.y + d13.x);
      const int tw = j * stride;                    // < N/4
      z[i0] = y0;                                   // sub-sequence k2 at i0 + k2 q
      z[i0 + q] = cmul(y1, __ldg(a.twiddle + tw));
      z[i0 + 2 * q] = cmul(y2, __ldg(a.twiddle + 2 * tw));
      const int t3 = 3 * tw;                        // may exceed N/2: use symmetry W^(N/2+x) = -W^x
      float2 w3 = t3 < (N >> 1) ? __ldg(a.twiddle + t3) : __ldg(a.twiddle + t3 - (N >> 1));
      if (t3 >= (N >> 1)) w3 = make_float2(-w3.x, -w3.y);
      z[i0 + 3 * q] = cmul(y3, w3);
    }
    len = q;
    lq -= 2;
    __syncthreads();
  }

  // epilogue: gather the crop, split the two real spectra, ramp, scale, store
  const int ma = ra / a.n_rx, mb = (ra + 1) / a.n_rx;
  const float sa = a.scale * (a.wsar ? __ldg(a.wsar + ma) : 1.f);
  const float sb = a.scale * (a.wsar ? __ldg(a.wsar + mb) : 1.f);
  float2* pa = a.prof + (size_t)ra * a.n_bins;
  float2* pb = pa + a.n_bins;
  for (int i = threadIdx.x; i < a.n_bins; i += BLOCK) {
    const int k = a.k_lo + i;
    const float2 Zk = z[digit_reverse(k, a.log2n)];
    const float2 Zn = z[digit_reverse((N - k) & (N - 1), a.log2n)];
    const float2 r = __ldg(a.ramp + i);
    // X_a = (Z[k] + conj Z[N-k]) / 2 ; X_b = (Z[k] - conj Z[N-k]) / (2j)
    const float2 A = make_float2(0.5f * (Zk.x + Zn.x), 0.5f * (Zk.y - Zn.y));
    const float2 B = make_float2(0.5f * (Zk.y + Zn.y), -0.5f * (Zk.x - Zn.x));
    const float2 Ar = cmul(A, r), Br = cmul(B, r);
    const bool in_spec = k <= (N >> 1);   // an even-length crop may end one bin past N/2 (A8: 0)
    pa[i] = in_spec ? make_float2(sa * Ar.x, sa * Ar.y) : make_float2(0.f, 0.f);
    if (has_b) pb[i] = in_spec ? make_float2(sb * Br.x, sb * Br.y) : make_float2(0.f, 0.f);
  }
}

}  // namespace

cudaError_t launch_rc(const RcArgs& a, cudaStream_t s) {
  constexpr int kBlock = 256;
  const size_t smem = (size_t)a.nfft * sizeof(float2);
  static std::atomic<bool> configured[kMaxDevices];   // the opt-in is per device
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if (!configured[dev].load()) {
    cudaError_t e = cudaFuncSetAttribute(rc_kernel<kBlock>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         16384 * (int)sizeof(float2));
    if (e != cudaSuccess) return e;
    configured[dev].store(true);
  }
  const int grid = (a.nrows + 1) / 2;
  rc_kernel<kBlock><<<grid, kBlock, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sar
