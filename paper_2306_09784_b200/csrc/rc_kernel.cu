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
#include <stdlib.h>

#include <algorithm>
#include <atomic>

#include "ptx_util.h"
#include "sar_internal.h"

#ifndef SAR_RC_MINB
#define SAR_RC_MINB 3
#endif

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

// ---------------------------------------------------------------------------------------
// rc_kernel_warp: the zero-padded transform as Zp = N / L transforms of length L (register
// path, L in {256, 512}, Ns <= L).  With x[t] = 0 for t >= L,
//   Z[Zp a + b] = sum_{t<L} (z[t] W_N^(b t)) W_L^(a t),      a < L, b < Zp,
// so warp b computes one L-point FFT of the pre-twiddled row pair entirely in registers,
// exchanging values between its radix-8 (last: radix-4 for L = 256) Stockham stages through
// its own row of shared memory with warp-level synchronisation only; the rows are then the
// b-major spectrum Z[Zp a + b] = Xs[b][a] the epilogue gathers the crop from.  One block-wide
// barrier per row pair (the classic kernel has one per radix-4 pass); shared-memory traffic
// per row pair about halves.  Numerically the same transform (fp32, fp64-built twiddles).
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 mul_mj(float2 a) { return make_float2(a.y, -a.x); }   // a * (-j)

// forward 4-point DFT, natural order in and out
__device__ __forceinline__ void dft4(float2& a0, float2& a1, float2& a2, float2& a3) {
  const float2 s02 = cadd(a0, a2), d02 = csub(a0, a2), s13 = cadd(a1, a3), d13 = mul_mj(csub(a1, a3));
  a0 = cadd(s02, s13);
  a2 = csub(s02, s13);
  a1 = cadd(d02, d13);
  a3 = csub(d02, d13);
}

// forward R-point DFT (R = 4 or 8) of v[0..R), natural order in and out
template <int R>
__device__ __forceinline__ void dft(float2* v) {
  if (R == 4) {
    dft4(v[0], v[1], v[2], v[3]);
  } else {
    constexpr float c = 0.70710678118654752f;
    // radix-2 split: even outputs from v[r] + v[r+4], odd outputs from (v[r] - v[r+4]) W_8^r
    float2 e[4], o[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      e[r] = cadd(v[r], v[r + 4]);
      o[r] = csub(v[r], v[r + 4]);
    }
    o[1] = make_float2(c * (o[1].x + o[1].y), c * (o[1].y - o[1].x));    // * (c, -c)
    o[2] = mul_mj(o[2]);                                                  // * -j
    o[3] = make_float2(c * (o[3].y - o[3].x), -c * (o[3].x + o[3].y));   // * (-c, -c)
    dft4(e[0], e[1], e[2], e[3]);
    dft4(o[0], o[1], o[2], o[3]);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      v[2 * m] = e[m];
      v[2 * m + 1] = o[m];
    }
  }
}

// physical index of entry i in a warp's row: one pad entry per 8 (conflict-free stride-8
// stage-0 stores and split-run stage-1 stores for 8-byte elements)
__device__ __forceinline__ int rpos(int i) { return i + (i >> 3); }

template <int L>
struct RcWarpPlan {
  static constexpr int E = L / 32;                 // values per lane
  static constexpr int RS = L + L / 8 + 2;         // row stride (complex): rows of different b
                                                   // start in different bank pairs
};

// One radix-R Stockham stage over a warp's row (NS = product of the radices before it):
// butterfly j takes in[j + r L/R], twiddles by W_(NS R)^((j mod NS) r), and writes its
// natural-order outputs to (j / NS) NS R + (j mod NS) + r NS.  Lane addresses are one base per
// butterfly plus compile-time offsets (rpos(i + 8 m) = rpos(i) + 9 m).  The twiddles are the
// powers w^r of the butterfly's base w = W_(NS R)^(j mod NS) (fp64-built, held in registers for
// the whole kernel), formed with at most three chained multiplications: loading R - 1 twiddles
// per butterfly from the plan table cost 23 % of the kernel's time (L1 wavefronts).
template <int R>
__device__ __forceinline__ void twiddle_powers(float2* v, const float2 w1) {
  float2 w[R];
  w[1] = w1;
#pragma unroll
  for (int r = 2; r < R; ++r) w[r] = (r % 2 == 0) ? cmul(w[r / 2], w[r / 2]) : cmul(w[r - 1], w1);
#pragma unroll
  for (int r = 1; r < R; ++r) v[r] = cmul(v[r], w[r]);
}

template <int L, int R, int NS>
__device__ __forceinline__ void stockham_stage(float2* v, float2* row, const float2* base, int lane) {
  constexpr int B = L / (32 * R);                  // butterflies per lane
  static_assert((L / R) % 8 == 0 && NS % 8 == 0, "stage offsets must be multiples of 8");
#pragma unroll
  for (int s = 0; s < B; ++s) {
    const float2* src = row + rpos(lane + 32 * s);
#pragma unroll
    for (int r = 0; r < R; ++r) v[s * R + r] = src[r * (L / R) * 9 / 8];
  }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < B; ++s) {
    twiddle_powers<R>(v + s * R, base[s]);
    dft<R>(v + s * R);
  }
#pragma unroll
  for (int s = 0; s < B; ++s) {
    const int j = lane + 32 * s;
    float2* dst = row + rpos((j / NS) * NS * R + (j % NS));
#pragma unroll
    for (int r = 0; r < R; ++r) dst[r * NS * 9 / 8] = v[s * R + r];
  }
  __syncwarp();
}

// Persistent CTAs: CTA c transforms row pairs c, c + grid, ...; with RING > 0 the raw rows of
// the next RING pairs are in flight into a shared-memory ring (one 1-D bulk copy of the pair's
// contiguous 2 Ns floats per stage, mbarrier completion), so the transform of one pair overlaps
// the HBM latency of the next ones.  RING = 0 reads the rows with plain loads (rows not 16-B
// aligned, or raw samples in mapped host memory).
// FULL: Ns == L (every BASELINE config at Ns = 512 or 256): stage 0 reads every sample with
// compile-time offsets, no clamp or zero select.
template <int L, int WARPS, int RING, bool FULL>
__global__ void __launch_bounds__(WARPS * 32, WARPS >= 8 ? SAR_RC_MINB : 1) rc_kernel_warp(const RcArgs a) {
  extern __shared__ __align__(16) float2 xs[];   // [zp][RS] | raw ring [RING][2 ns] | mbarriers
  constexpr int E = RcWarpPlan<L>::E, RS = RcWarpPlan<L>::RS;
  const int N = a.nfft;
  const int lzp = a.log2n - (L == 512 ? 9 : 8), zp = 1 << lzp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npairs = (a.nrows + 1) / 2;
  float* ring = reinterpret_cast<float*>(xs + zp * RS);
  const uint32_t bar0 = smem_u32(ring + RING * 2 * a.ns);
  auto issue = [&](int pair, int slot) {   // one thread: the pair's raw rows -> ring slot
    const int nr = min(2, a.nrows - 2 * pair);
    const uint32_t bytes = (uint32_t)(nr * a.ns) * 4u;
    mbar_arrive_expect_tx(bar0 + 8 * slot, bytes);
    bulk_g2s(smem_u32(ring + slot * 2 * a.ns), a.raw + (size_t)(a.row0 + 2 * pair) * a.ns, bytes, bar0 + 8 * slot);
  };
  if (RING > 0) {
    if (threadIdx.x == 0) {
      for (int d = 0; d < RING; ++d) mbar_init(bar0 + 8 * d, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int d = 0; d < RING; ++d)
        if (blockIdx.x + d * gridDim.x < npairs) issue(blockIdx.x + d * gridDim.x, d);
    }
    __syncthreads();
  }

  // twiddle bases of this lane's butterflies: stage 1 W_64^(j mod 8), stage 2 W_L^(j mod 64)
  constexpr int R2 = L / 64, B1 = L / (32 * 8), B2 = L / (32 * R2);
  float2 tw1[B1], tw2[B2];
#pragma unroll
  for (int s = 0; s < B1; ++s) tw1[s] = __ldg(a.stw + ((lane + 32 * s) % 8) * 8 + 1);
#pragma unroll
  for (int s = 0; s < B2; ++s) tw2[s] = __ldg(a.stw + 64 + ((lane + 32 * s) % 64) * R2 + 1);

  int it = 0;
  for (int pair = blockIdx.x; pair < npairs; pair += gridDim.x, ++it) {
    const int ra = a.row0 + 2 * pair;
    const bool has_b = 2 * pair + 1 < a.nrows;
    const float* xa;
    if (RING > 0) {
      constexpr int kR = RING > 0 ? RING : 1;   // (RING = 0 instantiations never take this branch)
      const int slot = it % kR;
      mbar_wait(bar0 + 8 * slot, (uint32_t)(it / kR) & 1u);
      xa = ring + slot * 2 * a.ns;
    } else {
      xa = a.raw + (size_t)ra * a.ns;
    }
    const float* xb = has_b ? xa + a.ns : xa;   // a lone last row reads row a again (unused)

    for (int b = warp; b < zp; b += WARPS) {
      float2 v[E];
      float2* row = xs + b * RS;
      const float2* cb = a.coef + (size_t)b * a.ns;
      // stage 0 (radix 8, no twiddles), one butterfly at a time; inputs
      // z[t] = c_b[t] (x_a[t] + j x_b[t]), c_b[t] = w[t] W_N^(b t), t = j + r L/8
#pragma unroll 1
      for (int s = 0; s < E / 8; ++s) {
        const int j = lane + 32 * s;
        // branch-free: all 24 loads of the butterfly are in flight together (a clamped index,
        // then zero for t >= Ns)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int t = j + r * (L / 8);
          const int tc = FULL ? t : min(t, a.ns - 1);
          const float2 c = __ldg(cb + tc);
          const float va = RING > 0 ? xa[tc] : __ldg(xa + tc);
          const float vb = has_b ? (RING > 0 ? xb[tc] : __ldg(xb + tc)) : 0.f;
          const float2 z = make_float2(c.x * va - c.y * vb, c.x * vb + c.y * va);
          v[r] = (FULL || t < a.ns) ? z : make_float2(0.f, 0.f);
        }
        dft<8>(v);
        float2* dst = row + 9 * j;                 // rpos(8 j + r) = 9 j + r
#pragma unroll
        for (int r = 0; r < 8; ++r) dst[r] = v[r];
      }
      __syncwarp();
      stockham_stage<L, 8, 8>(v, row, tw1, lane);
      stockham_stage<L, L / 64, 64>(v, row, tw2, lane);
    }
    __syncthreads();   // spectrum complete; the raw slot is consumed
    if (RING > 0 && threadIdx.x == 0 && pair + RING * (int)gridDim.x < npairs)
      issue(pair + RING * gridDim.x, it % (RING > 0 ? RING : 1));

    // epilogue as in rc_kernel, Z[k] = Xs[k mod zp][k / zp]
    const int ma = ra / a.n_rx, mb = (ra + 1) / a.n_rx;
    const float sa = a.scale * (a.wsar ? __ldg(a.wsar + ma) : 1.f);
    const float sb = a.scale * (a.wsar ? __ldg(a.wsar + mb) : 1.f);
    float2* pa = a.prof + (size_t)ra * a.n_bins;
    float2* pb = pa + a.n_bins;
    // Z[k] for k = k_lo + i and its mirror Z[N - k]; stepping i by the block (a multiple of zp)
    // keeps k mod zp and moves the row position by a constant: addresses advance linearly
    // (the crop lies in [0, N/2 + 1], so N - k never wraps except at k = 0)
    constexpr int kStep = WARPS * 32;
    const int hk = a.k_lo + threadIdx.x;
    const float2* zk = xs + (hk & (zp - 1)) * RS + rpos(hk >> lzp);
    const int hn = (N - hk) & (N - 1);
    const float2* zn = xs + (hn & (zp - 1)) * RS + rpos(hn >> lzp);
    const int dstep = rpos(kStep >> lzp);   // row positions per block step (kStep / zp is a multiple of 8)
    const bool lin = (kStep % zp) == 0 && ((kStep >> lzp) & 7) == 0 && a.k_lo > 0;
    // centring ramp exp(+j 2 pi k t_c / N): the table entry of the thread's first bin, then one
    // multiplication by the block step's ramp exp(+j 2 pi kStep t_c / N) per step (read from the
    // table as ramp[kStep] conj(ramp[0])): one load per thread instead of one per bin
    float2 rr = __ldg(a.ramp + min((int)threadIdx.x, a.n_bins - 1));
    float2 rstep = make_float2(1.f, 0.f);
    if (a.n_bins > kStep) {
      const float2 r0 = __ldg(a.ramp), rk = __ldg(a.ramp + kStep);
      rstep = make_float2(rk.x * r0.x + rk.y * r0.y, rk.y * r0.x - rk.x * r0.y);
    }
    for (int i = threadIdx.x; i < a.n_bins; i += kStep, zk += dstep, zn -= dstep, rr = cmul(rr, rstep)) {
      const int k = a.k_lo + i;
      float2 Zk, Zn;
      if (lin) {
        Zk = *zk;
        Zn = *zn;
      } else {
        const int kn = (N - k) & (N - 1);
        Zk = xs[(k & (zp - 1)) * RS + rpos(k >> lzp)];
        Zn = xs[(kn & (zp - 1)) * RS + rpos(kn >> lzp)];
      }
      const float2 r = rr;
      const float2 A = make_float2(0.5f * (Zk.x + Zn.x), 0.5f * (Zk.y - Zn.y));
      const float2 B = make_float2(0.5f * (Zk.y + Zn.y), -0.5f * (Zk.x - Zn.x));
      const float2 Ar = cmul(A, r), Br = cmul(B, r);
      const bool in_spec = k <= (N >> 1);
      pa[i] = in_spec ? make_float2(sa * Ar.x, sa * Ar.y) : make_float2(0.f, 0.f);
      if (has_b) pb[i] = in_spec ? make_float2(sb * Br.x, sb * Br.y) : make_float2(0.f, 0.f);
    }
    __syncthreads();   // the spectrum rows are free for the next pair
  }
}

#ifndef SAR_RC_RING
#define SAR_RC_RING 4
#endif
constexpr int kRcRing = SAR_RC_RING;

template <int L, int WARPS, int RING, bool FULL>
cudaError_t launch_warp_ring(const RcArgs& a, cudaStream_t s) {
  auto kern = rc_kernel_warp<L, WARPS, RING, FULL>;
  const size_t smem = (size_t)(a.nfft / L) * RcWarpPlan<L>::RS * sizeof(float2) +
                      (RING > 0 ? (size_t)RING * (2 * a.ns * sizeof(float) + 8) : 0);
  // the opt-in is per device: set once to the largest plan this instantiation can see
  // (N = 16384, Ns = L), so concurrent launches never lower it
  constexpr int kMaxSmem = (16384 / L) * RcWarpPlan<L>::RS * (int)sizeof(float2) +
                           (RING > 0 ? RING * (2 * L * (int)sizeof(float) + 8) : 0);
  static std::atomic<bool> configured[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if (!configured[dev].load()) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
    if (e != cudaSuccess) return e;
    configured[dev].store(true);
  }
  int resident = 0, sms = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, kern, WARPS * 32, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int npairs = (a.nrows + 1) / 2;
  const int grid = std::max(1, std::min(npairs, std::max(1, resident) * sms));
  kern<<<grid, WARPS * 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <int L, int WARPS>
cudaError_t launch_warp(const RcArgs& a, cudaStream_t s) {
  // bulk copies need 16-B aligned rows in device memory
  cudaPointerAttributes pa;
  const bool dev_mem = cudaPointerGetAttributes(&pa, a.raw) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
  const bool ring = dev_mem && a.ns % 4 == 0 && (reinterpret_cast<uintptr_t>(a.raw) & 15) == 0;
  if (!dev_mem) cudaGetLastError();   // clear a failed attribute query
  if (a.ns == L) return ring ? launch_warp_ring<L, WARPS, kRcRing, true>(a, s) : launch_warp_ring<L, WARPS, 0, true>(a, s);
  return ring ? launch_warp_ring<L, WARPS, kRcRing, false>(a, s) : launch_warp_ring<L, WARPS, 0, false>(a, s);
}

}  // namespace

// Which kernel transforms this plan's rows: the register path when the nonzero samples fit
// one L-point transform (L = 256 or 512), else the classic shared-memory FFT.
// SAR_RC_CLASSIC=1 forces the classic kernel (tests cover both).
int rc_path(int ns, int nfft, bool allow_env) {
  const char* e = allow_env ? getenv("SAR_RC_CLASSIC") : nullptr;
  if (e && e[0] == '1') return 0;
  if (ns <= 256 && nfft >= 256) return 256;
  if (ns <= 512 && nfft >= 512) return 512;
  return 0;
}

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
  const int L = rc_path(a.ns, a.nfft);
  if (L) {
    const int zp = a.nfft / L;
    if (L == 256) return zp >= 8 ? launch_warp<256, 8>(a, s) : zp >= 4 ? launch_warp<256, 4>(a, s)
                                 : zp >= 2 ? launch_warp<256, 2>(a, s) : launch_warp<256, 1>(a, s);
    return zp >= 8 ? launch_warp<512, 8>(a, s) : zp >= 4 ? launch_warp<512, 4>(a, s)
                   : zp >= 2 ? launch_warp<512, 2>(a, s) : launch_warp<512, 1>(a, s);
  }
  const int grid = (a.nrows + 1) / 2;
  rc_kernel<kBlock><<<grid, kBlock, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sar
