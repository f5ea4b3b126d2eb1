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

// Reverse the log2n-bit index in base 4 (with a leading base-2 digit when log2n is odd): DIF
// with a radix-2 first pass (if odd) then radix-4 passes leaves frequency k at position p =
// k with its mixed-radix digits [2 (if odd)], 4, ..., 4 reversed.  A base-4 digit reversal is
// the bit reversal with the two bits of every digit swapped back.
__device__ __forceinline__ int digit_reverse(int k, int log2n) {
  int p = 0, bits = log2n;
  if (log2n & 1) {            // the radix-2 digit is k's LSB and becomes p's MSB
    p = (k & 1) << (log2n - 1);
    k >>= 1;
    bits -= 1;
  }
  if (bits == 0) return p;
  unsigned r = __brev((unsigned)k) >> (32 - bits);
  r = ((r & 0x55555555u) << 1) | ((r >> 1) & 0x55555555u);
  return p | (int)r;
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) rc_kernel(const RcArgs a) {
  extern __shared__ float2 zs[];  // [nfft + nfft/32], padded
  // One pad slot per N/32 entries: the epilogue's digit-reversed gathers (32 bins whose
  // positions differ in their top five bits) then fall into distinct banks.
  const int sh = a.log2n > 5 ? a.log2n - 5 : 31;
#define Z(i) zs[(i) + ((i) >> sh)]
  const int N = a.nfft;
  const int ra = a.row0 + 2 * blockIdx.x;          // first row of the pair
  const bool has_b = 2 * blockIdx.x + 1 < a.nrows;
  const float* xa = a.raw + (size_t)ra * a.ns;
  const float* xb = xa + a.ns;

  int len = N;  // current sub-transform length
  int lq = a.log2n - (a.log2n & 1) - 2;            // log2 of the quarter length
  const float2 zero = make_float2(0.f, 0.f);
  if (!(a.log2n & 1) && a.ns <= (N >> 2)) {
    // Zero padding Z >= 4: the first radix-4 DIF pass sees x1 = x2 = x3 = 0 (they lie beyond Ns),
    // so its butterfly is y0 = y1 = y2 = y3 = x0; fuse it with the load:
    //   z[t + k N/4] = w[t] (x_a[t] + j x_b[t]) W_N^(k t),  k = 0..3
    const int q = N >> 2;
    for (int t = threadIdx.x; t < q; t += BLOCK) {
      float2 v = zero;
      if (t < a.ns) {
        const float w = __ldg(a.window + t);
        v.x = w * __ldg(xa + t);
        v.y = has_b ? w * __ldg(xb + t) : 0.f;
      }
      const float2 w1 = __ldg(a.twiddle + t);      // t < N/4
      const float2 w2 = cmul(w1, w1), w3 = cmul(w1, w2);
      Z(t) = v;
      Z(t + q) = cmul(v, w1);
      Z(t + 2 * q) = cmul(v, w2);
      Z(t + 3 * q) = cmul(v, w3);
    }
    len = q;
    lq -= 2;
    __syncthreads();
  } else {
    // load, window, zero-pad: z[t] = w[t] (x_a[t] + j x_b[t])
    for (int t = threadIdx.x; t < N; t += BLOCK) {
      float2 v = zero;
      if (t < a.ns) {
        const float w = __ldg(a.window + t);
        v.x = w * __ldg(xa + t);
        v.y = has_b ? w * __ldg(xb + t) : 0.f;
      }
      Z(t) = v;
    }
    __syncthreads();
    if (a.log2n & 1) {
      // radix-2 DIF pass over the whole array: pairs (i, i + N/2), twiddle W_N^i
      const int h = N >> 1;
      for (int i = threadIdx.x; i < h; i += BLOCK) {
        const float2 u = Z(i), v = Z(i + h);
        Z(i) = make_float2(u.x + v.x, u.y + v.y);
        Z(i + h) = cmul(make_float2(u.x - v.x, u.y - v.y), __ldg(a.twiddle + i));
      }
      len = h;
      __syncthreads();
    }
  }
  // radix-4 DIF passes: sub-transforms of length len, quarter q = len/4
  while (len >= 4) {
    const int q = len >> 2;
    const int stride = N / len;                    // twiddle index scale: W_len^j = W_N^(j*stride)
    const int nbf = N >> 2;                         // radix-4 butterflies per pass
    for (int b = threadIdx.x; b < nbf; b += BLOCK) {
      const int grp = b >> lq, j = b & (q - 1);
      const int i0 = (grp << (lq + 2)) + j;
      const float2 x0 = Z(i0), x1 = Z(i0 + q), x2 = Z(i0 + 2 * q), x3 = Z(i0 + 3 * q);
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
      const float2 w1 = __ldg(a.twiddle + tw);     // W^2 and W^3 by multiplication: one load
      const float2 w2 = cmul(w1, w1), w3 = cmul(w1, w2);
      Z(i0) = y0;                                   // sub-sequence k2 at i0 + k2 q
      Z(i0 + q) = cmul(y1, w1);
      Z(i0 + 2 * q) = cmul(y2, w2);
      Z(i0 + 3 * q) = cmul(y3, w3);
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
    const float2 Zk = Z(digit_reverse(k, a.log2n));
    const float2 Zn = Z(digit_reverse((N - k) & (N - 1), a.log2n));
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
  const size_t smem = (size_t)(a.nfft + (a.nfft >> 5) + 1) * sizeof(float2);   // padded (see rc_kernel)
  static std::atomic<bool> configured[kMaxDevices];   // the opt-in is per device
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if (!configured[dev].load()) {
    cudaError_t e = cudaFuncSetAttribute(rc_kernel<kBlock>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (16384 + 512 + 1) * (int)sizeof(float2));
    if (e != cudaSuccess) return e;
    configured[dev].store(true);
  }
  const int grid = (a.nrows + 1) / 2;
  rc_kernel<kBlock><<<grid, kBlock, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sar
