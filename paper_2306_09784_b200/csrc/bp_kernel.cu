// bp_kernel: tiled time-domain Back-Projection (steps H2-H6), Alg. 2 of arXiv 2306.09784
// in a form whose fp32 arithmetic is accurate at 30 m ranges.
//
// Work decomposition
//   * One CTA = one 32x32 pixel tile.  The tile anchor P_T is the tile centre (fp64).
//   * Warp NCW is the PRODUCER: for each ring stage of CB chirps it computes, in fp64,
//     the per-(tile, chirp, antenna) anchor record (D = P_T - q, r = |D|, anchor index
//     and anchor phase) and stages the W profile bins the tile can touch for that chirp
//     into shared memory in "pair" format {mid = (X[k]+X[k+1])/2, diff = X[k+1]-X[k]},
//     so that linear interpolation is one LDS.128 plus two FFMA.  The window bound is
//     the triangle inequality |d_hyp - d_anchor| <= 2 rho_T, valid for ANY track and
//     chirp order (no fallback path).
//   * Warps 0..NCW-1 are CONSUMERS: each thread owns PB pixels (register accumulators);
//     each warp's 32 lanes cover an 8x4 pixel patch so their gathers hit few bins.
//   * Producer/consumer hand-off through a kBpStages-deep ring guarded by mbarriers.
//
// Per (pixel, chirp, antenna) update (monostatic shown; bistatic adds the RX leg):
//   g   = D.u + |u|^2/2                      (u = p - P_T, fp32, |u| <= rho_T)
//   s   = r^2 + 2g  ~ |p - q|^2              rsqrt via MUFU: q = 1/sqrt(s)
//   R0  = s q;  t = R0 - r (exact);  h = (R0 + r)/2
//   dR  = t + (g - t h) q                     = |p - q| - r, to ~1e-8 m (one Newton step
//                                               on the residual; no cancellation)
//   kappa = kappa_anchor + A1 dR  (+ f_doppler(p))          Alg. 2 L8
//   phase = phi_anchor  + C2 dR                              Alg. 2 L9 (A2: +j)
//   v = mid[k] + (kappa - k - 1/2) diff[k],  k = round(kappa - 1/2) via the 1.5*2^23 trick
//   acc += v * exp(j phase)                   (MUFU sin/cos)  Alg. 2 L10, L12
// 3 MUFU + ~21 FMA/ALU + 1 LDS.128 per update.
#include <stdint.h>

#include "sar_internal.h"

namespace sar {
namespace {

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: x + kMagic rounds x to an integer
constexpr uint32_t kMagicBits = 0x4B400000u;
constexpr int kPatchX = 8, kPatchY = 4;  // pixel patch of one warp for one register slot

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

__device__ __forceinline__ float rsqrt_mufu(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One leg |p - q| - r of the anchored range (see header comment).
template <bool SAFE>
__device__ __forceinline__ float leg_delta(float Dx, float Dy, float r2, float r, float rh,
                                           float ux, float uy, float wh) {
  const float g = fmaf(Dx, ux, fmaf(Dy, uy, wh));
  if (SAFE) {
    // near field (an antenna may sit inside the tile): dR = 2g / (R + r), R = sqrt(max(s,0))
    const float s = fmaxf(fmaf(2.f, g, r2), 0.f);
    const float R = sqrtf(s);
    return __fdividef(2.f * g, R + r);
  } else {
    const float s = fmaf(2.f, g, r2);
    const float q = rsqrt_mufu(s);
    const float R0 = s * q;
    const float t = R0 - r;
    const float h = fmaf(R0, 0.5f, rh);
    const float rho = fmaf(-t, h, g);
    return fmaf(rho, q, t);
  }
}

// Shared-memory layout of one ring (all offsets in bytes, 16-B aligned):
//   [0, 64)                     mbarriers full[kBpStages], empty[kBpStages]
//   rec   [S][LEGS] x 32 B      monostatic: LEGS = items; bistatic: LEGS = CB + items
//   kwin  [S][items] int         window start bin per item (relative to the crop)
//   win   [S][items][W] x 16 B   pair-format profile windows
struct Layout {
  int items, legs;
  uint32_t rec, kwin, win, total;
};

__host__ __device__ inline Layout make_layout(int W, int CB, int n_rx, bool bistatic) {
  Layout L;
  L.items = CB * n_rx;
  L.legs = bistatic ? CB + L.items : L.items;
  L.rec = 64;
  L.kwin = L.rec + (uint32_t)kBpStages * L.legs * 32;
  uint32_t kw_bytes = ((uint32_t)kBpStages * L.items * 4 + 15u) & ~15u;
  L.win = L.kwin + kw_bytes;
  L.total = L.win + (uint32_t)kBpStages * L.items * W * 16;
  return L;
}

template <bool BISTATIC, bool DOP, bool SAFE, int NCW, int PB>
__global__ void __launch_bounds__((NCW + 1) * 32) bp_kernel(const BpArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Layout L = make_layout(a.W, a.CB, a.n_rx, BISTATIC);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase, bar_empty = sbase + 8 * kBpStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int tile = blockIdx.x;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int i0 = tx * kTileX;           // first grid column of the tile
  const int j0 = ty * kTileY;           // first row of the tile, relative to row0
  // tile anchor: centre of the full tile (even when ragged), fp64
  const double PTx = a.x0 + (i0 + 0.5 * (kTileX - 1)) * a.dx;
  const double PTy = a.y0 + (a.row0 + j0 + 0.5 * (kTileY - 1)) * a.dy;
  const double PTz = a.z0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kBpStages; ++s) {
      mbar_init(bar_full + 8 * s, 32);          // producer lanes
      mbar_init(bar_empty + 8 * s, NCW * 32);   // consumer threads
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int n_iter = (a.nchirp + a.CB - 1) / a.CB;

  if (warp == NCW) {
    // ============================== PRODUCER ==============================
    float4* rec = reinterpret_cast<float4*>(smem + L.rec);
    int* kwin = reinterpret_cast<int*>(smem + L.kwin);
    float4* win = reinterpret_cast<float4*>(smem + L.win);
    const double two_pi = 2.0 * kPi;
    for (int it = 0; it < n_iter; ++it) {
      const int slot = it % kBpStages;
      const uint32_t parity = (it / kBpStages) & 1;
      mbar_wait(bar_empty + 8 * slot, parity ^ 1);
      const int c0 = it * a.CB;
      const int cnt = min(a.CB, a.nchirp - c0);
      const int items = cnt * a.n_rx;
      float4* srec = rec + (size_t)slot * L.legs * 2;
      int* skw = kwin + slot * L.items;
      float4* swin = win + (size_t)slot * L.items * a.W;
      // ---- anchor records (fp64), one item per lane
      if (BISTATIC) {
        for (int c = lane; c < cnt; c += 32) {
          const double* q = a.tx + 3 * (size_t)(a.chirp0 + c0 + c);
          const double Dx = PTx - q[0], Dy = PTy - q[1], Dz = PTz - q[2];
          const float r = (float)sqrt(Dx * Dx + Dy * Dy + Dz * Dz);
          srec[2 * c] = make_float4((float)Dx, (float)Dy, r * r, r);
          srec[2 * c + 1] = make_float4(0.5f * r, 0.f, 0.f, 0.f);
        }
      }
      for (int e = lane; e < items; e += 32) {
        const int c = e / a.n_rx, n = e - c * a.n_rx;
        const int m = a.chirp0 + c0 + c;
        const double* qt = a.tx + 3 * (size_t)m;
        double d_anchor;
        float4 leg0;
        float rleg;
        if (BISTATIC) {
          const double* qr = a.rx + 3 * ((size_t)m * a.n_rx + n);
          const double Dx = PTx - qr[0], Dy = PTy - qr[1], Dz = PTz - qr[2];
          rleg = (float)sqrt(Dx * Dx + Dy * Dy + Dz * Dz);
          leg0 = make_float4((float)Dx, (float)Dy, rleg * rleg, rleg);
          const double Tx = PTx - qt[0], Ty = PTy - qt[1], Tz = PTz - qt[2];
          const float rt = (float)sqrt(Tx * Tx + Ty * Ty + Tz * Tz);
          d_anchor = (double)rt + (double)rleg;
        } else {
          const double Dx = PTx - qt[0], Dy = PTy - qt[1], Dz = PTz - qt[2];
          rleg = (float)sqrt(Dx * Dx + Dy * Dy + Dz * Dz);
          leg0 = make_float4((float)Dx, (float)Dy, rleg * rleg, rleg);
          d_anchor = 2.0 * (double)rleg;
        }
        const double kap = a.a1 * d_anchor - a.k_lo;               // anchor index in the crop
        const int k0 = (int)floor(kap - a.kap_half) - 1;            // window start
        double ph = a.c2 * d_anchor;                                // anchor phase (cycles)
        ph -= rint(ph);
        const uint32_t waddr = smem_u32(swin + (size_t)e * a.W);
        const uint32_t off = waddr - 16u * kMagicBits;
        const int ri = BISTATIC ? a.CB + e : e;
        srec[2 * ri] = leg0;
        srec[2 * ri + 1] = make_float4(0.5f * rleg, (float)(kap - k0 - 0.5), (float)(two_pi * ph),
                                       __uint_as_float(off));
        skw[e] = k0;
      }
      __syncwarp();
      // ---- profile windows in pair format; 8 items per batch for memory-level parallelism
      for (int j0w = 0; j0w < a.W; j0w += 31) {
        for (int e0 = 0; e0 < items; e0 += 8) {
          float2 x[8];
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            x[b] = make_float2(0.f, 0.f);
            const int e = e0 + b;
            if (e < items) {
              const int c = e / a.n_rx, n = e - c * a.n_rx;
              const size_t row = ((size_t)(a.chirp0 + c0 + c) * a.n_rx + n) * a.n_bins;
              const int k = skw[e] + j0w + lane;
              if (k >= 0 && k < a.n_bins) x[b] = __ldg(a.prof + row + k);
            }
          }
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            const float nx_ = __shfl_down_sync(0xffffffffu, x[b].x, 1);
            const float ny_ = __shfl_down_sync(0xffffffffu, x[b].y, 1);
            const int e = e0 + b;
            const int j = j0w + lane;
            if (e < items && lane < 31 && j < a.W) {
              swin[(size_t)e * a.W + j] =
                  make_float4(0.5f * (x[b].x + nx_), 0.5f * (x[b].y + ny_), nx_ - x[b].x, ny_ - x[b].y);
            }
          }
        }
      }
      mbar_arrive(bar_full + 8 * slot);
    }
    return;
  }

  // ============================== CONSUMERS ==============================
  const int lx = lane & (kPatchX - 1), ly = lane >> 3;
  constexpr int kPatchesPerRow = kTileX / kPatchX;
  float ux[PB], uy[PB], wh[PB], acc_r[PB], acc_i[PB], fd[PB];
  int gx[PB], gy[PB];
#pragma unroll
  for (int p = 0; p < PB; ++p) {
    const int pi = warp * PB + p;
    const int xl = (pi % kPatchesPerRow) * kPatchX + lx;
    const int yl = (pi / kPatchesPerRow) * kPatchY + ly;
    gx[p] = i0 + xl;
    gy[p] = j0 + yl;
    const double dux = (xl - 0.5 * (kTileX - 1)) * a.dx;
    const double duy = (yl - 0.5 * (kTileY - 1)) * a.dy;
    ux[p] = (float)dux;
    uy[p] = (float)duy;
    wh[p] = (float)(0.5 * (dux * dux + duy * duy));
    acc_r[p] = 0.f;
    acc_i[p] = 0.f;
    fd[p] = 0.f;
    if (DOP) {
      if (gx[p] < a.nx && gy[p] < a.nrow) fd[p] = __ldg(a.dop + (size_t)(a.row0 + gy[p]) * a.nx + gx[p]);
    }
    // keep the per-pixel constants in registers: a shuffle is opaque to ptxas, which
    // otherwise re-derives them from fp64 inside the chirp loop (rematerialisation)
    ux[p] = __shfl_sync(0xffffffffu, ux[p], lane);
    uy[p] = __shfl_sync(0xffffffffu, uy[p], lane);
    wh[p] = __shfl_sync(0xffffffffu, wh[p], lane);
  }
  const float4* rec = reinterpret_cast<const float4*>(smem + L.rec);
  const float A1 = a.A1f, C2 = a.C2f;

  for (int it = 0; it < n_iter; ++it) {
    const int slot = it % kBpStages;
    const uint32_t parity = (it / kBpStages) & 1;
    mbar_wait(bar_full + 8 * slot, parity);
    const int cnt = min(a.CB, a.nchirp - it * a.CB);
    const float4* srec = rec + (size_t)slot * L.legs * 2;
    if (!BISTATIC) {
#pragma unroll 1
      for (int c = 0; c < cnt; ++c) {
        const float4 A = srec[2 * c], B = srec[2 * c + 1];
        const uint32_t off = __float_as_uint(B.w);
#pragma unroll
        for (int p = 0; p < PB; ++p) {
          const float dR = leg_delta<SAFE>(A.x, A.y, A.z, A.w, B.x, ux[p], uy[p], wh[p]);
          float kap = fmaf(A1, dR, B.y);
          if (DOP) kap += fd[p];
          const float ph = fmaf(C2, dR, B.z);
          const float tk = kap + kMagic;
          const float kf = tk - kMagic;
          const float gf = kap - kf;
          const float4 e = lds128(__float_as_uint(tk) * 16u + off);
          const float vr = fmaf(gf, e.z, e.x), vi = fmaf(gf, e.w, e.y);
          float sn, cs;
          __sincosf(ph, &sn, &cs);
          acc_r[p] = fmaf(vr, cs, acc_r[p]);
          acc_r[p] = fmaf(-vi, sn, acc_r[p]);
          acc_i[p] = fmaf(vr, sn, acc_i[p]);
          acc_i[p] = fmaf(vi, cs, acc_i[p]);
        }
      }
    } else {
#pragma unroll 1
      for (int c = 0; c < cnt; ++c) {
        const float4 T = srec[2 * c], TB = srec[2 * c + 1];
        float dT[PB];
#pragma unroll
        for (int p = 0; p < PB; ++p) dT[p] = leg_delta<SAFE>(T.x, T.y, T.z, T.w, TB.x, ux[p], uy[p], wh[p]);
#pragma unroll 1
        for (int n = 0; n < a.n_rx; ++n) {
          const int ri = a.CB + c * a.n_rx + n;
          const float4 A = srec[2 * ri], B = srec[2 * ri + 1];
          const uint32_t off = __float_as_uint(B.w);
#pragma unroll
          for (int p = 0; p < PB; ++p) {
            const float dR = dT[p] + leg_delta<SAFE>(A.x, A.y, A.z, A.w, B.x, ux[p], uy[p], wh[p]);
            float kap = fmaf(A1, dR, B.y);
            if (DOP) kap += fd[p];
            const float ph = fmaf(C2, dR, B.z);
            const float tk = kap + kMagic;
            const float kf = tk - kMagic;
            const float gf = kap - kf;
            const float4 e = lds128(__float_as_uint(tk) * 16u + off);
            const float vr = fmaf(gf, e.z, e.x), vi = fmaf(gf, e.w, e.y);
            float sn, cs;
            __sincosf(ph, &sn, &cs);
            acc_r[p] = fmaf(vr, cs, acc_r[p]);
            acc_r[p] = fmaf(-vi, sn, acc_r[p]);
            acc_i[p] = fmaf(vr, sn, acc_i[p]);
            acc_i[p] = fmaf(vi, cs, acc_i[p]);
          }
        }
      }
    }
    mbar_arrive(bar_empty + 8 * slot);
  }

  // epilogue: store (or accumulate) the tile
#pragma unroll
  for (int p = 0; p < PB; ++p) {
    if (gx[p] < a.nx && gy[p] < a.nrow) {
      float2* dst = a.img + (size_t)gy[p] * a.nx + gx[p];
      if (a.accumulate) {
        const float2 o = *dst;
        *dst = make_float2(o.x + acc_r[p], o.y + acc_i[p]);
      } else {
        *dst = make_float2(acc_r[p], acc_i[p]);
      }
    }
  }
}

constexpr int kNCW = 8;   // consumer warps
constexpr int kPB = 4;    // pixels per consumer thread
static_assert(kNCW * kPB * kPatchX * kPatchY == kTileX * kTileY, "tile / warp map mismatch");

template <bool BI, bool DOP, bool SAFE>
cudaError_t launch_one(const BpArgs& a, cudaStream_t s) {
  auto kern = bp_kernel<BI, DOP, SAFE, kNCW, kPB>;
  const Layout L = make_layout(a.W, a.CB, a.n_rx, BI);
  static int configured_bytes = -1;
  if ((int)L.total > configured_bytes) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess) return e;
    configured_bytes = (int)L.total;
  }
  const int tiles_y = (a.nrow + kTileY - 1) / kTileY;
  const long grid = (long)a.tiles_x * tiles_y;
  kern<<<(unsigned)grid, (kNCW + 1) * 32, L.total, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

size_t bp_smem_bytes(int W, int CB, int n_rx, bool bistatic) {
  return make_layout(W, CB, n_rx, bistatic).total;
}

cudaError_t launch_bp(const BpArgs& a, bool bistatic, bool doppler, bool safe, cudaStream_t s) {
  if (bistatic) {
    if (doppler) return safe ? launch_one<true, true, true>(a, s) : launch_one<true, true, false>(a, s);
    return safe ? launch_one<true, false, true>(a, s) : launch_one<true, false, false>(a, s);
  }
  if (doppler) return safe ? launch_one<false, true, true>(a, s) : launch_one<false, true, false>(a, s);
  return safe ? launch_one<false, false, true>(a, s) : launch_one<false, false, false>(a, s);
}

}  // namespace sar
