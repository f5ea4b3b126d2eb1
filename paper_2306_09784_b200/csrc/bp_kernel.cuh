// bp_kernel.cuh: the tiled Back-Projection kernel template (steps H2-H6), included by
// bp_kernel.cu (plain epilogue: store / accumulate / chirp-split reductions into the image)
// and bp_scatter.cu (NEXT-4 scatter epilogue into peer images), so that the two families are
// compiled as separate translation units and the plain kernel's code is not perturbed by the
// scatter epilogue (ptxas schedules the chirp loop differently when it is present: +2.5 % C3).
#pragma once
// bp_kernel: tiled time-domain Back-Projection (steps H2-H6), Alg. 2 of arXiv 2306.09784
// in a form whose fp32 arithmetic is accurate at 30 m ranges.
//
// Work decomposition
//   * One CTA = one 32 x (NCW*PB) pixel tile.  The tile anchor P_T is the tile centre (fp64).
//   * Warp NCW is the PRODUCER: for each ring stage of CB chirps it computes, in fp64,
//     the per-(tile, chirp, antenna) anchor record (D = P_T - q, r = |D|, anchor index
//     and anchor phase) and stages the W profile entries the tile can touch for that chirp
//     into shared memory in "pair" format {mid = (X[k]+X[k+1])/2, diff = X[k+1]-X[k]} x
//     carrier bin phase, so that linear interpolation is one LDS.128 plus two FFMA.  The
//     entries come from pair-format rows built once per chirp row (pair_kernel) with one
//     1-D bulk copy (TMA engine) per item; without that workspace the producer builds them
//     itself from the profiles (same values; the path used if the rows cannot be allocated).
//     The window bound is the triangle inequality |d_hyp - d_anchor| <= 2 rho_T (tighter
//     for polar tiles), valid for ANY track and chirp order.
//   * Warps 0..NCW-1 are CONSUMERS: each thread owns PB pixels (register accumulators);
//     for one register slot a warp's 32 lanes cover an 8x4 pixel patch, so their gathers
//     hit few distinct bins (broadcast, no bank conflicts).
//   * Producer/consumer hand-off through an S-deep ring guarded by mbarriers
//     (full: 32 producer lanes arrive; empty: all consumer threads arrive).
//
// Per (pixel, chirp, antenna) update (monostatic shown; bistatic adds the RX leg):
//   g   = D.u + |u|^2/2                      (u = p - P_T, fp32, |u| <= rho_T)
//   s   = r^2 + 2g  ~ |p - q|^2              rsqrt via MUFU: q = 1/sqrt(s)
//   R0  = s q;  t = R0 - r (exact);  h = (R0 + r)/2
//   dR  = t + (g - t h) q                     = |p - q| - r, to ~1e-8 m (one Newton step
//                                               on the residual; no cancellation)
//   kappa = kappa_anchor + A1 dR  (+ f_doppler(p))          Alg. 2 L8
//   K = floor(kappa) (the 1.5*2^23 trick), f = kappa - K, gf = f - 1/2
//   v = mid[K] + gf diff[K]                   (one LDS.128, two FFMA)
//   acc += v * exp(j 2 pi beta gf)            (MUFU sin/cos)  Alg. 2 L9, L10, L12
// Carrier phase folding: without Doppler kappa = a1 d exactly, so the hypothetical
// phase 2 pi c2 d (Alg. 2 L9, A2: +j) equals 2 pi beta kappa with beta = c2/a1 cycles per
// bin = 2 pi beta (K + 1/2) + 2 pi beta gf.  The producer multiplies each staged pair by
// exp(j 2 pi beta (K + 1/2)) (plan table, built in fp64), so the per-update MUFU argument
// is bounded by |2 pi beta gf| <= pi beta (~32 rad) whatever the range: the fp32 phase
// carries no bias that grows with range or tile size.  With Doppler the shift
// exp(-j 2 pi beta f_doppler(p)) is a per-pixel constant applied in the epilogue.
// 3 MUFU + ~21 FMA/ALU + 1 LDS.128 per update.
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <type_traits>

#include "ptx_util.h"
#include "sar_internal.h"

namespace sar {
namespace {

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: x + kMagic rounds x to an integer
#ifndef SAR_BP_NRX_SPEC
// derived bistatic stages with a compile-time RX count (0: off), for the 4-RX MIMO radar of the
// paper's Measure F and config C4: C4 rank shard 124.2 -> 121.0 ms
#define SAR_BP_NRX_SPEC 4
#endif
#ifndef SAR_BP_GROUP
#define SAR_BP_GROUP 8
#endif
#ifndef SAR_BP_JUNROLL
#define SAR_BP_JUNROLL 8
#endif
constexpr int kGroup = SAR_BP_GROUP;     // derived-chirp group (monostatic): one rsqrt per group
constexpr int kJUnroll = SAR_BP_JUNROLL;
#ifndef SAR_BP_DERIVE_MONO
#define SAR_BP_DERIVE_MONO 1
#endif
#ifndef SAR_BP_DERIVE_BI
#define SAR_BP_DERIVE_BI 1
#endif
#ifndef SAR_BP_COL_MONO
// collinear monostatic groups (tuning switch): fewer FFMA2 per derived chirp, but the extra
// group variants cost registers and spills -- measured slower on C0/C2 (straight) and C3
// (9.42 -> 9.86, 21.50 -> 22.04, 52.13 -> 52.93 ms); the bistatic stages keep them (C4 -2 %)
#define SAR_BP_COL_MONO 0
#endif
constexpr bool kColMono = SAR_BP_COL_MONO;
#ifndef SAR_BP_HORNER
// derived legs in Horner form in E: R_b (sqrt(1 + E Q^2) - 1) = E (Q/2 + E (-Q^3/8 + E (Q^5/16 ..)))
// with the coefficients formed once per group / stage (one FFMA2 per term instead of E Q, delta,
// P(delta), EQ P)
#define SAR_BP_HORNER 1
#endif
#ifndef SAR_BP_HORNER_MAX
#define SAR_BP_HORNER_MAX 2   // Horner form for series of at most this many terms (measured: 2 -> C3 -0.6 %; 3-4 term Horner variants cost registers: C3 +1.9 %, C4 shard +0 to +19 %)
#endif
constexpr bool kHorner = SAR_BP_HORNER;
constexpr int kHornerMax = SAR_BP_HORNER_MAX;
#ifndef SAR_BP_HORNER_MAX_BI
// bistatic stages (3-4 terms) in Horner form too, at three resident CTAs per SM (72 registers):
// C4 rank shard 118.7-120.5 -> 115.65 ms, C6 10.36 -> 9.87 ms (tools/gpu_r4i.sh); at four CTAs
// (56 registers) the extra coefficients spilled (+14-19 %)
#define SAR_BP_HORNER_MAX_BI 4
#endif
constexpr int kHornerMaxBi = SAR_BP_HORNER_MAX_BI;
constexpr bool kDeriveMono = SAR_BP_DERIVE_MONO;   // derived-chirp groups compiled in (monostatic)
constexpr bool kDeriveBi = SAR_BP_DERIVE_BI;       // derived stages compiled in (bistatic)
// Derived legs (reading A22): R sqrt(1 + delta) - R by the binomial series truncated after t
// terms; the Taylor remainder bounds the truncation by R |delta|^(t+1) c_t (1 - |delta|)^-(t+1/2)
// with c_2 = 1/16, c_3 = 5/128, c_4 = 7/256.  A group (stage) takes the fewest terms whose bound,
// evaluated in fp64 over the whole tile (R <= r_b + rho_T + |o|), stays below kTruncMax; with
// none, every leg keeps its own rsqrt.  kTruncMax = 1e-9 m is ~3e-6 rad of carrier phase per
// update, 10x below the fp32 rounding of a leg (~1e-8 m).
constexpr double kTruncMax = 1e-9;
constexpr double kDeltaMax = 0.05;   // (and |delta| small enough that the remainder factor is ~1)
// fewest series terms (2..tmax) of a leg with |delta| <= dl at range <= R; 99: not derivable
__device__ __forceinline__ int series_terms(double dl, double R, int tmin, int tmax) {
  if (!(dl >= 0.0 && dl <= kDeltaMax)) return 99;
  const double f = 1.0 / (1.0 - dl);
  double p = R * dl * dl * dl * f * f * sqrt(f);   // R dl^3 (1 - dl)^-2.5
  const double c[3] = {1.0 / 16.0, 5.0 / 128.0, 7.0 / 256.0};
  for (int t = 2; t <= 4; ++t, p *= dl * f) {
    if (t >= tmin && t <= tmax && c[t - 2] * p <= kTruncMax) return t;
  }
  return 99;
}
// Collinear legs: pixels lie in the plane z = z0, so a leg's offset o enters the per-pixel part of
// E = -2 (D_b + u).o + |o|^2 through its horizontal part only.  When every horizontal offset of a
// group (stage) lies along one unit direction e -- a straight track, an array along it -- then
// o_h.u = (o_h.e)(e.u) and the consumers spend one FFMA2 on E (e.u formed once per group).  The
// dropped perpendicular part changes a leg by <= |o_perp| rho_T / (r_b - rho_T): a group is
// collinear when that stays below kTruncMax / 10.
// group_dir: e = direction of the largest horizontal offset among `width` aligned lanes (xor
// butterfly, ties broken lexicographically so that every lane ends with the same vector).
__device__ __forceinline__ void group_dir(double ox, double oy, int width, double& ex, double& ey) {
  double n = ox * ox + oy * oy, bx = ox, by = oy;
  for (int s = 1; s < width; s <<= 1) {
    const double n2 = __shfl_xor_sync(0xffffffffu, n, s), x2 = __shfl_xor_sync(0xffffffffu, bx, s),
                 y2 = __shfl_xor_sync(0xffffffffu, by, s);
    if (n2 > n || (n2 == n && (x2 > bx || (x2 == bx && y2 > by)))) {
      n = n2;
      bx = x2;
      by = y2;
    }
  }
  const double len = sqrt(n);
  ex = len > 0.0 ? bx / len : 1.0;
  ey = len > 0.0 ? by / len : 0.0;
}
__device__ __forceinline__ bool leg_collinear(double ox, double oy, double ex, double ey, double rho, double rmin) {
  return fabs(ox * ey - oy * ex) * rho <= 0.1 * kTruncMax * rmin;
}
constexpr uint32_t kMagicBits = 0x4B400000u;
constexpr int kPatchX = 8, kPatchY = 4;  // pixel patch of one warp for one register slot
#ifndef SAR_BP_BATCH
#define SAR_BP_BATCH 8
#endif
constexpr int kBatch = SAR_BP_BATCH;     // producer: profile rows loaded per batch
#ifndef SAR_BP_CHIRP_UNROLL
#define SAR_BP_CHIRP_UNROLL 1            // consumer chirp-loop unroll (monostatic)
#endif
constexpr int kChirpUnroll = SAR_BP_CHIRP_UNROLL;
#ifndef SAR_BP_MIN_SPLIT
#define SAR_BP_MIN_SPLIT 256               // chirp split: (chirp, RX) items per chunk at least
#endif
constexpr long kMinSplitItems = SAR_BP_MIN_SPLIT;
#ifndef SAR_BP_SPLIT_WAVES
// chirp split: aim for this many waves of resident CTAs.  Beyond filling the GPU, chirp chunks
// shorten the tail wave and make the CTAs resident at one time stream fewer distinct pair rows
// through L2 (chunk-major order); measured (tools/libsweep.sh) 8 -> 32 waves: C3 58.94 -> 58.73 ms,
// C0 10.08 -> 9.94, C2 24.14 -> 23.83, C6 11.42 -> 11.22, C6p 1.522 -> 1.499 ms
#define SAR_BP_SPLIT_WAVES 32
#endif
constexpr long kSplitWaves = SAR_BP_SPLIT_WAVES;
// Scatter launches (the fused gather; sar_form_image's host-image stores) aim at 16 waves and never
// run unsplit: measured on one GPU (tools/rank_probe2.py, tools/scatter_policy.sh), per-rank C3 tile
// blocks N = 2: 28.44 ms unsplit (7.5 waves) -> 27.80 split; N = 8: 7.13 (32 waves) -> 7.09; C3 e2e
// (host image) 56.62 -> 55.86 ms
constexpr long kScatterWaves = 16;
#ifndef SAR_BP_L2_WINDOW_MB
#define SAR_BP_L2_WINDOW_MB 64   // pair-row bytes of one chirp chunk at most (126 MB L2 on two dies)
#endif
constexpr long kL2WindowMB = SAR_BP_L2_WINDOW_MB;
constexpr long kScatterUnsplit = 1L << 40;   // (a depth at which a scatter would run unsplit: none)
inline long env_long(const char* name, long dflt) {
  const char* e = getenv(name);
  return e && *e ? atol(e) : dflt;
}
// pixel (column x, image row y) inside the launch's image rows (y < 0: a tile row starting above)
#define SAR_PIX_OK(x, y) ((x) < a.nx && (unsigned)(y) < (unsigned)a.nrow)
#ifndef SAR_BP_RX_UNROLL
#define SAR_BP_RX_UNROLL 4                // bistatic RX-loop unroll (C4 1146 -> 1112 ms; 2 is slower)
#endif
constexpr int kRxUnroll = SAR_BP_RX_UNROLL;
// (A min-blocks launch bound, even "1", changes ptxas's schedule: measured 5 % slower on C3;
//  capping registers for 6-7 resident CTAs spilled and was slower too.  tools/vsweep.sh)

#ifdef SAR_BP_TRACE
// tuning instrumentation (tools/trace_bp.py): clock64 stamps of the ring waits of four CTAs
constexpr int kTrCtas = 4, kTrIt = 256;
__device__ unsigned long long g_trace[kTrCtas][9][kTrIt][3];
__device__ unsigned int g_trace_wid[kTrCtas][9][2];
__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int tr_cta() {
  const int b = blockIdx.x;
  return b == 2000 ? 0 : b == 2001 ? 1 : b == 5000 ? 2 : b == 5001 ? 3 : -1;
}
__device__ __forceinline__ void tr_ids(int trc, int w) {
  unsigned int wid, smid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  g_trace_wid[trc][w][0] = wid;
  g_trace_wid[trc][w][1] = smid;
}
#define SAR_TR(w, it, k) \
  if (trc >= 0 && lane == 0 && (it) < kTrIt) g_trace[trc][w][it][k] = clk()
#else
#define SAR_TR(w, it, k)
#endif

#ifdef SAR_DEBUG_CHECKS
// bounds-check build (tools/check_cases.py): violations counted per kind, read back through
// sar_debug_violations_*: [0] consumer window index outside its item's W entries, [1] chirp-chunk
// workspace plane out of range, [2] pair-row bulk copy outside its row (clamped), [3] consumer
// read outside the shared-memory allocation
__device__ unsigned long long g_violations[4];
#define SAR_CHECK(cond, k) \
  if (!(cond)) atomicAdd(&g_violations[k], 1ull)
// derived-leg modes built by the producers (tests: every mode exercised): [0] mono 2-term group,
// [1] mono 3-term, [2] / [3] mono collinear 2 / 3 terms, [4] bistatic 3-term stage, [5] 4-term,
// [6] / [7] bistatic collinear 3 / 4 terms
__device__ unsigned long long g_modes[8];
#define SAR_MODE(k) atomicAdd(&g_modes[k], 1ull)
#else
#define SAR_CHECK(cond, k)
#define SAR_MODE(k)
#endif

__device__ __forceinline__ unsigned ctaid_x() {   // opaque to CSE: not kept live across loops
  unsigned v;
  asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(v));
  return v;
}

// window entry address of rounded index bits tk (1.5 * 2^23 + K): 16 B per entry from `off`
// (one IMAD; written as shift + add, ptxas emits the same IMAD)
__device__ __forceinline__ uint32_t win_addr(float tk, uint32_t off) { return __float_as_uint(tk) * 16u + off; }

__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

// Packed fp32 pairs (sm_100 FFMA2 / FADD2 / FMUL2): one instruction, two round-to-nearest
// fp32 operations.  A pair whose halves are equal is issued as a scalar broadcast operand,
// so record values are read once for two pixels (the BP loop is register-file-read bound).
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float lo2(f32x2 v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return a;
}
__device__ __forceinline__ float hi2(f32x2 v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return b;
}
__device__ __forceinline__ f32x2 ffma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f32x2 fadd2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 fsub2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 fmul2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 bc2(float a) { return pk2(a, a); }

// Horner coefficients of the series, Q ~ 1/R_b: H[0] = Q/2, H[1] = -Q^3/8, H[2] = Q^5/16, H[3] = -5 Q^7/128
template <int TERMS>
__device__ __forceinline__ void horner_coef(const f32x2 Q, f32x2* H) {
  const f32x2 Q2 = fmul2(Q, Q);
  H[0] = fmul2(Q, bc2(0.5f));
  H[1] = fmul2(fmul2(Q2, Q), bc2(-0.125f));
  if (TERMS >= 3) H[2] = fmul2(fmul2(Q2, H[1]), bc2(-0.5f));
  if (TERMS >= 4) H[3] = fmul2(fmul2(Q2, H[2]), bc2(-0.625f));
}
// base + E (H0 + E (H1 + E (H2 + E H3)))
template <int TERMS>
__device__ __forceinline__ f32x2 horner_leg(const f32x2 E, const f32x2* H, const f32x2 base) {
  f32x2 t = H[TERMS - 1];
#pragma unroll
  for (int k = TERMS - 2; k >= 0; --k) t = ffma2(E, t, H[k]);
  return ffma2(E, t, base);
}

__device__ __forceinline__ float rsqrt_mufu(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One leg |p - q| - r of the anchored range.  Record: Dx, Dy, r2 = r^2, r, e = r/2 (fast)
// or Dz^2 (SAFE).  SAFE is the near-field form (an antenna may sit inside the tile): the
// range is formed from the exact differences D + u and dR = 2g / (R + r) has no division
// by a vanishing quantity (r > 0: the anchor is never a pixel centre).
//   D2x, D2y = 2 D (record), w = |u|^2 (per pixel): g2 = 2 D.u + |u|^2 = |D + u|^2 - r^2
//   s = r^2 + g2, q = rsqrt(s); t = s q - r and H = s q + r (one rounding each);
//   rho2 = g2 - t H = s - (s q)^2 (exact residual up to one rounding);
//   dR = t + rho2 q / 2.
template <bool SAFE>
__device__ __forceinline__ float leg_delta(float D2x, float D2y, float r2, float r, float dz2,
                                           float ux, float uy, float w) {
  const float g2 = fmaf(D2x, ux, fmaf(D2y, uy, w));
  if (SAFE) {
    const float ex = fmaf(0.5f, D2x, ux), ey = fmaf(0.5f, D2y, uy);
    const float R = sqrtf(fmaf(ex, ex, fmaf(ey, ey, dz2)));
    return __fdividef(g2, R + r);
  } else {
    const float s = g2 + r2;
    const float q = rsqrt_mufu(s);
    const float t = fmaf(s, q, -r);
    const float H = fmaf(s, q, r);
    const float qh = 0.5f * q;
    const float rho2 = fmaf(-t, H, g2);
    return fmaf(rho2, qh, t);
  }
}

// The far-field leg for a pixel pair (FFMA2 form of leg_delta<false>); record
// A = {2Dx, 2Dy, r^2, r}; the second record word is B = {kappa_anchor, window address,
// Dz^2 (near field), 0}, so the consumer reads (kappa_anchor, address) with one LDS.64.
__device__ __forceinline__ f32x2 leg_delta2(const float4 A, const f32x2 UX, const f32x2 UY, const f32x2 W) {
  const f32x2 G2 = ffma2(bc2(A.x), UX, ffma2(bc2(A.y), UY, W));   // 2 D.u + |u|^2
  const f32x2 S = fadd2(G2, bc2(A.z));                            // ~|p - q|^2
  const f32x2 Q = pk2(rsqrt_mufu(lo2(S)), rsqrt_mufu(hi2(S)));
  const f32x2 T = ffma2(S, Q, bc2(-A.w));                         // s q - r
  const f32x2 H = ffma2(S, Q, bc2(A.w));                          // s q + r
  const f32x2 RHO = ffma2(pk2(-lo2(T), -hi2(T)), H, G2);          // exact residual
  return ffma2(RHO, fmul2(Q, bc2(0.5f)), T);                      // |p - q| - r
}

// Antenna phase centre as the producer uses it.  Polar plans bound each tile's window by the
// declared antenna box (tighter than the triangle inequality): a position outside the box is
// clamped into it, so a false declaration gives wrong values but every window read stays in
// range.  Cartesian windows hold for any position (triangle inequality): used as given.
struct Q3 {
  double x, y, z;
};
__device__ __forceinline__ Q3 ld_pos(const double* q, const BpArgs& a) {
  Q3 r{q[0], q[1], q[2]};
  if (a.polar) {
    r.x = fmin(fmax(r.x, a.box_lo[0]), a.box_hi[0]);
    r.y = fmin(fmax(r.y, a.box_lo[1]), a.box_hi[1]);
    r.z = fmin(fmax(r.z, a.box_lo[2]), a.box_hi[2]);
  }
  return r;
}

// leg_delta2 that also returns Q = rsqrt(s) ~ 1/|p - q| (derived-chirp groups)
__device__ __forceinline__ f32x2 leg_delta2q(const float4 A, const f32x2 UX, const f32x2 UY, const f32x2 W, f32x2& Q) {
  const f32x2 G2 = ffma2(bc2(A.x), UX, ffma2(bc2(A.y), UY, W));
  const f32x2 S = fadd2(G2, bc2(A.z));
  Q = pk2(rsqrt_mufu(lo2(S)), rsqrt_mufu(hi2(S)));
  const f32x2 T = ffma2(S, Q, bc2(-A.w));
  const f32x2 H = ffma2(S, Q, bc2(A.w));
  const f32x2 RHO = ffma2(pk2(-lo2(T), -hi2(T)), H, G2);
  return ffma2(RHO, fmul2(Q, bc2(0.5f)), T);
}

// Shared-memory layout (bytes, 16-B aligned):
//   [0, 128)                     mbarriers full[kBpMaxStages], empty[kBpMaxStages]
//   [128, 160)                   producer scratch
//   rec   [S][LEGS] x 32 B       monostatic: LEGS = items; bistatic: LEGS = CB + items
//   kwin  [S][items] int2        {window start bin (crop-relative), profile row}
//   win   [S][items][W] x 16 B   pair-format profile windows
struct Layout {
  int items, legs;
  uint32_t flags, rec, kwin, win, total;
};

__host__ __device__ inline Layout make_layout(int W, int CB, int n_rx, int S, bool bistatic) {
  Layout L;
  L.items = CB * n_rx;
  L.legs = bistatic ? CB + L.items : L.items;
  L.flags = 16 * kBpMaxStages;   // producer scratch (derived-group flags of the stage being built)
  L.rec = L.flags + 32;
  L.kwin = L.rec + (uint32_t)S * L.legs * 32;
  const uint32_t kw_bytes = ((uint32_t)S * L.items * 8 + 15u) & ~15u;
  L.win = L.kwin + kw_bytes;
  L.total = L.win + (uint32_t)S * L.items * W * 16;
  return L;
}

// NEAR: the plan has tiles within 3 rho of the antenna box; those tiles (a per-CTA,
// warp-uniform decision) take the near-field SAFE consumer path, all others the fast one.
template <bool BISTATIC, bool DOP, bool NEAR, int NCW, int PB, bool SCATTER>
__device__ __forceinline__ void bp_body(const BpArgs& a) {
  constexpr int TX = kTileX;
  constexpr int TY = NCW * PB * kPatchX * kPatchY / kTileX;
  extern __shared__ __align__(16) unsigned char smem[];
  const int S = a.S;
  const Layout L = make_layout(a.W, a.CB, a.n_rx, S, BISTATIC);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase, bar_empty = sbase + 8 * kBpMaxStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // CTA -> (chirp chunk, tile), chunk-major so that concurrently resident CTAs stream the
  // same profile rows through L2.  Tiles are ABSOLUTE grid tiles (tile = ty * tiles_x + tx of the
  // whole grid, range [tile0, tile0 + ntile)): every pixel is computed with the same anchor
  // whatever the shard, so a row or tile shard reproduces the unsharded image (Alg. 2's pixel
  // loop is independent per pixel).  ksplit > 1 for grids too small to fill
  // the GPU (chunks summed in chunk order: deterministic).
  // The launch covers whole tile rows [ty0, ty0 + ntile / tiles_x); CTAs outside the valid
  // launch-local range [tile_lo, tile_hi) (a tile shard's ragged first / last tile row) exit
  // at once.  (This form of the index arithmetic, launch-local with the row offset added last,
  // keeps ptxas's fastest schedule of the chirp loop: adding an absolute tile offset before
  // the division by tiles_x measured 2.7 % slower on C3.)
  const unsigned tile_l = blockIdx.x % (unsigned)a.ntile, chunk = blockIdx.x / (unsigned)a.ntile;
  if (tile_l < (unsigned)a.tile_lo || tile_l >= (unsigned)a.tile_hi) return;
  const int chirp0 = a.chirp0 + (int)chunk * a.chunk;
  const int nchirp = min(a.chunk, a.nchirp - (int)chunk * a.chunk);
  const int tx = (int)(tile_l % (unsigned)a.tiles_x), ty = (int)(tile_l / (unsigned)a.tiles_x) + a.ty0;
  const int i0 = tx * TX;               // first grid column of the tile
  const int J0 = ty * TY;               // first grid row of the tile (absolute)
  const int j0 = J0 - a.row0;           // ... relative to the image's first row (may be < 0)
  // tile anchor: centre of the full tile (even when ragged), fp64.  Cartesian grids:
  // (x0 + i dx, y0 + j dy); polar grids (Measure E): (xc + r sin th, yc + r cos th).
  double PTx, PTy;
  if (a.polar) {
    const double th = a.th0 + (i0 + 0.5 * (TX - 1)) * a.dth;
    const double rr = a.r0 + (J0 + 0.5 * (TY - 1)) * a.dr;
    PTx = a.x0 + rr * sin(th);
    PTy = a.y0 + rr * cos(th);
  } else {
    PTx = a.x0 + (i0 + 0.5 * (TX - 1)) * a.dx;
    PTy = a.y0 + (J0 + 0.5 * (TY - 1)) * a.dy;
  }
  const double PTz = a.z0;
  // near-field test of this tile (NEAR kernels): distance from the anchor to the antenna box;
  // rho_t = the tile's half-diagonal (polar: farthest corner from the anchor)
  double rho_t = a.tile_rho;
  if (a.polar) {   // annular patch: farthest from its anchor at a corner
    const double rc = a.r0 + (J0 + 0.5 * (TY - 1)) * a.dr;
    const double ht = 0.5 * (TX - 1) * a.dth, hr = 0.5 * (TY - 1) * a.dr;
    rho_t = 0.0;
    for (int c = 0; c < 4; ++c) {
      const double rr = rc + ((c & 1) ? hr : -hr), dt = (c & 2) ? ht : -ht;
      rho_t = fmax(rho_t, sqrt(rr * rr + rc * rc - 2.0 * rr * rc * cos(dt)));
    }
  }
  bool tile_near = false;
  if constexpr (NEAR) {
    double d2 = 0.0;
    const double pt[3] = {PTx, PTy, PTz};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double gap = fmax(0.0, fmax(a.box_lo[k] - pt[k], pt[k] - a.box_hi[k]));
      d2 += gap * gap;
    }
    const double near_r = 3.0 * rho_t * (1.0 + 1e-6) + 1e-3;
    tile_near = d2 < near_r * near_r;
  }
  // derived-chirp groups: far-field monostatic tiles of plans that allow them
  // (derived stages only in the default 8 x 4 bistatic shape: in the 4 x 4 polar shape the extra
  //  code alone costs registers and measured 20 % on C6p, whose short stages gain nothing)
#ifndef SAR_BP_DERBI_44
#define SAR_BP_DERBI_44 0
#endif
  constexpr bool kDerBi = kDeriveBi && ((NCW == 8 && PB == 4) || (SAR_BP_DERBI_44 && NCW == 4 && PB == 4));
  const bool derive = kDeriveMono && !BISTATIC && a.derive && !tile_near;
  const bool derive_bi = kDerBi && BISTATIC && a.derive && !tile_near;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(bar_full + 8 * s, 32);          // producer lanes
      mbar_init(bar_empty + 8 * s, NCW * 32);   // consumer threads
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int n_iter = (nchirp + a.CB - 1) / a.CB;

  if (warp == NCW) {
    // ============================== PRODUCER ==============================
    float4* rec = reinterpret_cast<float4*>(smem + L.rec);
    int2* kwin = reinterpret_cast<int2*>(smem + L.kwin);
    float4* win = reinterpret_cast<float4*>(smem + L.win);
    int slot = 0;
    uint32_t parity = 0;
#ifdef SAR_BP_TRACE
    const int trc = tr_cta();
    if (trc >= 0 && lane == 0) tr_ids(trc, 8);
#endif
    for (int it = 0; it < n_iter; ++it) {
      SAR_TR(8, it, 0);
      mbar_wait(bar_empty + 8 * slot, parity ^ 1);
      SAR_TR(8, it, 1);
      const int c0 = it * a.CB;
      const int cnt = min(a.CB, nchirp - c0);
      const int items = cnt * a.n_rx;
      float4* srec = rec + (size_t)slot * L.legs * 2;
      int2* skw = kwin + slot * L.items;
      float4* swin = win + (size_t)slot * L.items * a.W;
      // ---- anchor records (fp64), one item per lane
      if (BISTATIC) {
        for (int c = lane; c < cnt; c += 32) {
          const Q3 q = ld_pos(a.tx + 3 * (size_t)(chirp0 + c0 + c), a);
          const double Dx = PTx - q.x, Dy = PTy - q.y, Dz = PTz - q.z;
          const float r = (float)sqrt(Dx * Dx + Dy * Dy + Dz * Dz);
          srec[2 * c] = make_float4((float)(2.0 * Dx), (float)(2.0 * Dy), r * r, r);
          srec[2 * c + 1] = make_float4(0.f, 0.f, NEAR ? (float)(Dz * Dz) : 0.f, 0.f);
        }
      }
      for (int e = lane; e < items; e += 32) {
        const int c = BISTATIC ? e / a.n_rx : e;
        const int n = BISTATIC ? e - c * a.n_rx : 0;
        const int m = chirp0 + c0 + c;
        const Q3 qt = ld_pos(a.tx + 3 * (size_t)m, a);
        // The consumers form r32 + dR = sqrt(r32^2 + 2 D32.u + |u|^2) from the fp32-rounded
        // record; the anchor path length uses the exact fp64 |D| so that the rounding of
        // r and D enters only at second order (|r32 - |D|| * dR / r, ~1e-8 m).
        double d_anchor, dz;
        float4 leg0;
        float rleg;
        if (BISTATIC) {
          const Q3 qr = ld_pos(a.rx + 3 * ((size_t)m * a.n_rx + n), a);
          const double Dx = PTx - qr.x, Dy = PTy - qr.y, Dz = PTz - qr.z;
          const double rr = sqrt(Dx * Dx + Dy * Dy + Dz * Dz);
          rleg = (float)rr;
          leg0 = make_float4((float)(2.0 * Dx), (float)(2.0 * Dy), rleg * rleg, rleg);
          dz = Dz;
          const double Tx = PTx - qt.x, Ty = PTy - qt.y, Tz = PTz - qt.z;
          d_anchor = sqrt(Tx * Tx + Ty * Ty + Tz * Tz) + rr;
        } else {
          const double Dx = PTx - qt.x, Dy = PTy - qt.y, Dz = PTz - qt.z;
          const double rr = sqrt(Dx * Dx + Dy * Dy + Dz * Dz);
          rleg = (float)rr;
          leg0 = make_float4((float)(2.0 * Dx), (float)(2.0 * Dy), rleg * rleg, rleg);
          dz = Dz;
          d_anchor = 2.0 * rr;
        }
        const double kap = a.a1 * d_anchor - a.k_lo;               // anchor index in the crop
        const int k0 = (int)floor(kap - a.kap_half) - 1;            // window start
        const int wh = a.W >> 1;                                    // centre the fp32 index
        const uint32_t waddr = smem_u32(swin + (size_t)e * a.W);
        const uint32_t off = waddr + 16u * (uint32_t)wh - 16u * kMagicBits;
        const int ri = BISTATIC ? a.CB + e : e;
        srec[2 * ri] = leg0;
        srec[2 * ri + 1] = make_float4((float)(kap - k0 - 0.5 - wh), __uint_as_float(off),
                                       NEAR ? (float)(dz * dz) : 0.f, 0.f);
        skw[e] = make_int2(k0, m * a.n_rx + n);   // profile row (size_t offsets below: rows x n_bins may exceed 2^31)
      }
      if (BISTATIC && derive_bi && cnt >= 4) {   // (short stages: the base leg does not amortise)
        // Derived stage (bistatic): every leg of the stage -- the TX legs of chirps 1.. and all
        // RX legs -- follows from chirp 0's TX leg (the stage base b) by the series of the
        // monostatic groups, with o = q_leg - q_tx(b) (RX offsets included), so the consumers
        // spend one rsqrt per pixel per stage.  Records: TX of chirp c >= 1 and every RX item
        // {-2 o_x, -2 o_y, -2 D_b.o + |o|^2, -}.  Series terms (3 or 4) per stage: the most any
        // leg needs, |delta| <= (2 (r_b + rho_T) |o| + |o|^2) / (r_b - rho_T)^2 (series_terms).
        // Anchor indices: every RX leg's at 2 r_b (windows their own), split as
        // kappa_b - 1/2 = n + phi with n an integer: the record holds n - k0 - W/2 + 1.5 2^23
        // (exact in fp32) and the base record the fraction eps = phi / A1 (metres), which the
        // consumers add to the base leg, so that the rounding of the index is one FFMA2.
        const Q3 qb = ld_pos(a.tx + 3 * (size_t)(chirp0 + c0), a);
        const double Dbx = PTx - qb.x, Dby = PTy - qb.y, Dbz = PTz - qb.z;
        const double rb = sqrt(Dbx * Dbx + Dby * Dby + Dbz * Dbz), rmin = rb - rho_t;
        auto leg_o = [&](int k, double& ox, double& oy, double& oz) {   // k < items: RX item, else TX chirp
          const Q3 q = ld_pos(k < items ? a.rx + 3 * ((size_t)(chirp0 + c0) * a.n_rx + k)
                                        : a.tx + 3 * (size_t)(chirp0 + c0 + (k - items)), a);
          ox = q.x - qb.x;
          oy = q.y - qb.y;
          oz = q.z - qb.z;
        };
        int tneed = 2;
        double mx = 0.0, my = 0.0;   // this lane's largest horizontal offset
        for (int k = lane; k < items + cnt; k += 32) {
          double ox, oy, oz;
          leg_o(k, ox, oy, oz);
          const double on = sqrt(ox * ox + oy * oy + oz * oz);
          const double dl = rmin > 0.0 ? (2.0 * (rb + rho_t) * on + on * on) / (rmin * rmin) : -1.0;
          tneed = max(tneed, series_terms(dl, rb + rho_t + on, 3, 4));
          if (ox * ox + oy * oy > mx * mx + my * my) {
            mx = ox;
            my = oy;
          }
        }
        tneed = __reduce_max_sync(0xffffffffu, tneed);
        double ex, ey;
        group_dir(mx, my, 32, ex, ey);
        bool col = true;
        for (int k = lane; k < items + cnt; k += 32) {
          double ox, oy, oz;
          leg_o(k, ox, oy, oz);
          col = col && leg_collinear(ox, oy, ex, ey, rho_t, rmin);
        }
        col = __all_sync(0xffffffffu, col);
        __syncwarp();   // the stage's records (other lanes) are complete
        if (tneed <= 4) {
          const double kb = a.a1 * 2.0 * rb - a.k_lo - 0.5, nb = floor(kb);
          const int wh = a.W >> 1;
          for (int k = lane; k < items + cnt; k += 32) {
            if (k == items) continue;   // chirp 0's TX leg stays the base leg
            double ox, oy, oz;
            leg_o(k, ox, oy, oz);
            const double cj = -2.0 * (Dbx * ox + Dby * oy + Dbz * oz) + (ox * ox + oy * oy + oz * oz);
            // collinear records are {s, c, nM, window address}: one LDS.128 per RX leg
            const float nM = (float)(nb - skw[k < items ? k : 0].x - wh + (double)kMagic);
            const float4 rec_o = col ? make_float4((float)(-2.0 * (ox * ex + oy * ey)), (float)cj, nM,
                                                   k < items ? srec[2 * (a.CB + k) + 1].y : 0.f)
                                     : make_float4((float)(-2.0 * ox), (float)(-2.0 * oy), (float)cj, 0.f);
            if (k < items) {
              srec[2 * (a.CB + k)] = rec_o;
              srec[2 * (a.CB + k) + 1].x = nM;
            } else {
              srec[2 * (k - items)] = rec_o;
            }
          }
          if (lane == 0) SAR_MODE(4 + (tneed - 3) + (col ? 2 : 0));
          if (lane == 0)   // chirp 0's TX record: {e, eps, terms (+ 16: collinear)}
            srec[1] = make_float4((float)ex, (float)ey, (float)((kb - nb) / (double)a.A1f), (float)(tneed + (col ? 16 : 0)));
        }
        __syncwarp();
      }
      if (!BISTATIC && derive) {
        // Derived-chirp groups (monostatic): within a group of kGroup consecutive chirps of the
        // stage, chirp j's range follows from the group base b's by the convergent series
        //   |p - q_j| = R_b sqrt(1 + delta),  delta = E / R_b^2,
        //   E = |p - q_j|^2 - |p - q_b|^2 = -2 (D_b + u).o + |o|^2,  o = q_j - q_b, D_b = P_T - q_b,
        // so the consumers spend one rsqrt per pixel per group instead of per chirp.  The record
        // of a derived chirp is {-2 o_x, -2 o_y, c = -2 D_b.o + |o|^2 (fp64 -> fp32), -} and its
        // anchor index is taken at the base's anchor distance (its window start is its own).  A
        // group is derived only when the series bound holds over the whole tile with 2 or 3 terms
        // (series_terms), |delta| <= (2 (r_b + rho_T) |o| + |o|^2) / (r_b - rho_T)^2 (any track,
        // any chirp order: otherwise every chirp of the group keeps its own leg).  As in the
        // bistatic stages, the group's anchor indices are integers + 1.5 2^23 and the base record
        // carries the fraction eps = phi / A1 (z) and the series terms (w).
        __syncwarp();
        const int wh = a.W >> 1;
        for (int e0 = 0; e0 < items; e0 += 32) {
          const int c = e0 + lane;
          const int cb = c - (c % kGroup);
          int t = 99;
          double ox = 0, oy = 0, oz = 0, Dbx = 0, Dby = 0, Dbz = 0, rb = 0;
          if (c < cnt && cb + kGroup <= cnt) {
            const Q3 qj = ld_pos(a.tx + 3 * (size_t)(chirp0 + c0 + c), a);
            const Q3 qb = ld_pos(a.tx + 3 * (size_t)(chirp0 + c0 + cb), a);
            ox = qj.x - qb.x;
            oy = qj.y - qb.y;
            oz = qj.z - qb.z;
            Dbx = PTx - qb.x;
            Dby = PTy - qb.y;
            Dbz = PTz - qb.z;
            rb = sqrt(Dbx * Dbx + Dby * Dby + Dbz * Dbz);
            const double on = sqrt(ox * ox + oy * oy + oz * oz), rmin = rb - rho_t;
            if (rmin > 0.0) t = series_terms((2.0 * (rb + rho_t) * on + on * on) / (rmin * rmin), rb + rho_t + on, 2, 3);
          }
          // the group's terms: the most any of its kGroup lanes needs
          int tg = t;
#pragma unroll
          for (int s = 1; s < kGroup; s <<= 1) tg = max(tg, __shfl_xor_sync(0xffffffffu, tg, s));
          // collinear group (e from the group's largest offset; records 1 and 2 carry e in w)
          double ex = 1.0, ey = 0.0;
          bool col = false;
          if constexpr (kColMono) {
            group_dir(ox, oy, kGroup, ex, ey);
            const unsigned cbal = __ballot_sync(0xffffffffu, leg_collinear(ox, oy, ex, ey, rho_t, rb - rho_t));
            col = ((cbal >> (lane & ~(kGroup - 1))) & ((1u << kGroup) - 1)) == ((1u << kGroup) - 1);
          }
          if (c < cnt && tg <= 3) {
            const double kb = a.a1 * 2.0 * rb - a.k_lo - 0.5, nb = floor(kb);
            srec[2 * c + 1].x = (float)(nb - skw[c].x - wh + (double)kMagic);
            if (c == cb) SAR_MODE((tg - 2) + (col ? 2 : 0));
            if (c == cb) {   // base record: the group is derived with tg terms (+ 4: collinear)
              srec[2 * c + 1].z = (float)((kb - nb) / (double)a.A1f);
              srec[2 * c + 1].w = (float)(tg + (col ? 4 : 0));
            } else {
              const double cj = -2.0 * (Dbx * ox + Dby * oy + Dbz * oz) + (ox * ox + oy * oy + oz * oz);
              const int j = c - cb;
              srec[2 * c] = col ? make_float4((float)(-2.0 * (ox * ex + oy * ey)), 0.f, (float)cj,
                                              j == 1 ? (float)ex : j == 2 ? (float)ey : 0.f)
                                : make_float4((float)(-2.0 * ox), (float)(-2.0 * oy), (float)cj, 0.f);
            }
          }
        }
      }
      __syncwarp();
      if (a.pairs) {
        // bulk copies of pair-format rows: lane 0 adds the stage's byte count to the full
        // barrier, every lane arrives after issuing its copies; a start outside the padded row
        // (antennas outside the declared box) is clamped: wrong values, never out of bounds
        if (lane == 0) mbar_arrive_expect_tx(bar_full + 8 * slot, (uint32_t)items * a.W * 16u);
        __syncwarp();
        const uint32_t wdst = smem_u32(swin);
        for (int e = lane; e < items; e += 32) {
          const int2 kw = skw[e];
          SAR_CHECK(kw.x + a.pair_pad >= 0 && kw.x + a.pair_pad <= a.pair_stride - a.W, 2);
          const int i0 = min(max(kw.x + a.pair_pad, 0), a.pair_stride - a.W);
          bulk_g2s(wdst + 16u * (uint32_t)(e * a.W), a.pairs + (size_t)kw.y * a.pair_stride + i0, 16u * a.W,
                   bar_full + 8 * slot);
        }
        if (lane != 0) mbar_arrive(bar_full + 8 * slot);
        SAR_TR(8, it, 2);
        if (++slot == S) {
          slot = 0;
          parity ^= 1;
        }
        continue;
      }
      // ---- profile windows in pair format: lane j of an item produces entry j from bins
      //      k0+j and k0+j+1 (the latter from lane j+1 by shuffle); kBatch rows in flight
      for (int j0w = 0; j0w < a.W; j0w += 31) {
        const int j = j0w + lane;
        for (int e0 = 0; e0 < items; e0 += kBatch) {
          float2 x[kBatch];
#pragma unroll
          for (int b = 0; b < kBatch; ++b) {
            x[b] = make_float2(0.f, 0.f);
            const int e = e0 + b;
            if (e < items) {
              const int2 kw = skw[e];
              const int k = kw.x + j;
              if (k >= 0 && k < a.n_bins) x[b] = __ldg(a.prof + (size_t)kw.y * a.n_bins + k);
            }
          }
#pragma unroll
          for (int b = 0; b < kBatch; ++b) {
            const float nx_ = __shfl_down_sync(0xffffffffu, x[b].x, 1);
            const float ny_ = __shfl_down_sync(0xffffffffu, x[b].y, 1);
            const int e = e0 + b;
            if (e < items && lane < 31 && j < a.W) {
              // bin phase exp(j 2 pi beta (k_lo + k + 1/2)) of the entry's lower bin k; the
              // table starts at k = -1 (the entry holding X[-1] = 0 and X[0]); entries
              // further out hold only zeros and may take any phase
              const int k = min(max(skw[e].x + j, -1), a.n_bins - 1);
              const float2 q = __ldg(a.binphase + k + 1);
              const float mr = 0.5f * (x[b].x + nx_), mi = 0.5f * (x[b].y + ny_);
              const float dr = nx_ - x[b].x, di = ny_ - x[b].y;
              swin[(size_t)e * a.W + j] = make_float4(mr * q.x - mi * q.y, mr * q.y + mi * q.x,
                                                      dr * q.x - di * q.y, dr * q.y + di * q.x);
            }
          }
        }
      }
      mbar_arrive(bar_full + 8 * slot);
      SAR_TR(8, it, 2);
      if (++slot == S) {
        slot = 0;
        parity ^= 1;
      }
    }
    return;
  }

  // ============================== CONSUMERS ==============================
  auto consume = [&](auto safe_tag) {
  constexpr bool SAFE = decltype(safe_tag)::value;
  const int lx = lane & (kPatchX - 1), ly = lane >> 3;
  constexpr int kPatchesPerRow = TX / kPatchX;
  float ux[PB], uy[PB], wh[PB], acc_r[PB], acc_i[PB], fd[PB];
  int gx[PB], gy[PB];
#pragma unroll
  for (int p = 0; p < PB; ++p) {
    const int pi = warp * PB + p;
    const int xl = (pi % kPatchesPerRow) * kPatchX + lx;
    const int yl = (pi / kPatchesPerRow) * kPatchY + ly;
    gx[p] = i0 + xl;
    gy[p] = j0 + yl;
    double dux, duy;
    if (a.polar) {   // pixel offset from the anchor, both evaluated in fp64
      const double th = a.th0 + (i0 + xl) * a.dth;
      const double rr = a.r0 + (J0 + yl) * a.dr;
      dux = (a.x0 + rr * sin(th)) - PTx;
      duy = (a.y0 + rr * cos(th)) - PTy;
    } else {
      dux = (xl - 0.5 * (TX - 1)) * a.dx;
      duy = (yl - 0.5 * (TY - 1)) * a.dy;
    }
    ux[p] = (float)dux;
    uy[p] = (float)duy;
    wh[p] = (float)(dux * dux + duy * duy);   // |u|^2
    acc_r[p] = 0.f;
    acc_i[p] = 0.f;
    fd[p] = 0.f;
    if (DOP) {
      // clamped to the plan's declared bound: a table exceeding it gives wrong values for those
      // pixels, never a read outside the staged window
      if (SAR_PIX_OK(gx[p], gy[p]))
        fd[p] = fminf(fmaxf(__ldg(a.dop + (size_t)(J0 + yl) * a.nx + gx[p]), -a.dop_max), a.dop_max);
    }
    // keep the per-pixel constants in registers: a shuffle is opaque to ptxas, which
    // otherwise re-derives them from fp64 inside the chirp loop (rematerialisation)
    ux[p] = __shfl_sync(0xffffffffu, ux[p], lane);
    uy[p] = __shfl_sync(0xffffffffu, uy[p], lane);
    wh[p] = __shfl_sync(0xffffffffu, wh[p], lane);
  }
  const float4* rec = reinterpret_cast<const float4*>(smem + L.rec);
  const float A1 = a.A1f, C3 = a.C3f;
  constexpr bool kPaired = !SAFE && (PB % 2 == 0);
  f32x2 UX[PB / 2 + 1], UY[PB / 2 + 1], W2[PB / 2 + 1], FD2[PB / 2 + 1], ACC[PB + 1], ACI[PB + 1];
  if (kPaired) {
#pragma unroll
    for (int h = 0; h < PB / 2; ++h) {
      UX[h] = pk2(ux[2 * h], ux[2 * h + 1]);
      UY[h] = pk2(uy[2 * h], uy[2 * h + 1]);
      W2[h] = pk2(wh[2 * h], wh[2 * h + 1]);
      FD2[h] = pk2(fd[2 * h], fd[2 * h + 1]);
    }
#pragma unroll
    for (int p = 0; p < PB; ++p) ACC[p] = ACI[p] = pk2(0.f, 0.f);
  }

  int slot = 0;
  uint32_t parity = 0;
#ifdef SAR_BP_TRACE
  const int trc = tr_cta();
  if (trc >= 0 && lane == 0) tr_ids(trc, warp);
#endif
  for (int it = 0; it < n_iter; ++it) {
    SAR_TR(warp, it, 0);
    mbar_wait(bar_full + 8 * slot, parity);
    SAR_TR(warp, it, 1);
    const int cnt = min(a.CB, nchirp - it * a.CB);
    const float4* srec = rec + (size_t)slot * L.legs * 2;
    if (kPaired) {
      // Far field, pixels in pairs (2h, 2h+1): the range and index arithmetic runs as
      // FFMA2/FADD2 over the pair with the record values as scalar broadcast operands; the
      // complex interpolation and accumulation run as FFMA2 over (re, im).
      // v exp(j th) = vr (cs, sn) + vi (-sn, cs): the two halves go to separate accumulators,
      // ACC += vr (cs, sn) and ACI += vi (sn, cs) (a swizzle, no negation); the epilogue
      // forms (ACC.re - ACI.re, ACC.im + ACI.im).
      // tail_core: TK = 1.5 2^23 + round(kappa) (its bits address the window entry), GF = kappa -
      // round(kappa) in [-1/2, 1/2]
      auto tail_core = [&](const int h, const f32x2 TK, const f32x2 GF, const uint32_t off) {
        const f32x2 TH = fmul2(GF, bc2(C3));                                        // 2 pi beta gf
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const float tk = k ? hi2(TK) : lo2(TK);
          const float gf = k ? hi2(GF) : lo2(GF);
          SAR_CHECK((unsigned)((int)(__float_as_uint(tk) - kMagicBits) + (a.W >> 1)) < (unsigned)a.W, 0);
          SAR_CHECK(__float_as_uint(tk) * 16u + off >= sbase + L.win &&
                    __float_as_uint(tk) * 16u + off + 16u <= sbase + L.total, 3);
          const float4 e = lds128(win_addr(tk, off));
          const f32x2 V = ffma2(bc2(gf), pk2(e.z, e.w), pk2(e.x, e.y));             // lerp (re, im)
          float sn, cs;
          __sincosf(k ? hi2(TH) : lo2(TH), &sn, &cs);
          ACC[2 * h + k] = ffma2(bc2(lo2(V)), pk2(cs, sn), ACC[2 * h + k]);
          ACI[2 * h + k] = ffma2(bc2(hi2(V)), pk2(sn, cs), ACI[2 * h + k]);
        }
      };
      // tail: the leg's own anchor index kap_a (fractional)                       Alg. 2 L8
      auto tail = [&](const int h, const f32x2 DR, const float kap_a, const uint32_t off) {
        f32x2 KAP = ffma2(bc2(A1), DR, bc2(kap_a));
        if (DOP) KAP = fadd2(KAP, FD2[h]);
        const f32x2 TK = fadd2(KAP, bc2(kMagic));                                   // round
        tail_core(h, TK, fsub2(KAP, fsub2(TK, bc2(kMagic))), off);
      };
      // tail_n: derived legs, whose DR carries the anchor's fraction (eps) and whose record holds
      // the integer rest nM = n + 1.5 2^23: TK = A1 DR + nM is the rounding, nM - TK is exact
      auto tail_n = [&](const int h, const f32x2 DR, const float nM, const uint32_t off) {
        if (DOP) {
          const f32x2 KF = ffma2(bc2(A1), DR, FD2[h]);
          const f32x2 TK = fadd2(KF, bc2(nM));
          tail_core(h, TK, fadd2(KF, fsub2(bc2(nM), TK)), off);
        } else {
          const f32x2 TK = ffma2(bc2(A1), DR, bc2(nM));
          tail_core(h, TK, ffma2(bc2(A1), DR, fsub2(bc2(nM), TK)), off);
        }
      };
      if (!BISTATIC) {
        for (int c = 0; c < cnt;) {
          const float4 A = srec[2 * c], B = srec[2 * c + 1];
          if (kDeriveMono && B.w != 0.f) {
            // derived group (warp-uniform: one record for all): the base chirp's leg (plus the
            // anchor fraction eps = B.z), then the kGroup - 1 others by the series
            //   |p - q_j| - r_b = dR_b + (E Q) P(delta),  delta = E Q^2 (Q = 1/R_b),
            //   P = 1/2 - delta/8 (+ delta^2/16 with 3 terms, B.w = 3)
            f32x2 DR0[PB / 2], Q0[PB / 2];
#pragma unroll
            for (int h = 0; h < PB / 2; ++h) {
              DR0[h] = fadd2(leg_delta2q(A, UX[h], UY[h], W2[h], Q0[h]), bc2(B.z));
              tail_n(h, DR0[h], B.x, __float_as_uint(B.y));
            }
            auto group = [&](auto terms_tag, auto col_tag) {
              constexpr int TERMS = decltype(terms_tag)::value;
              constexpr bool COL = decltype(col_tag)::value;   // collinear: E = c + s (e.u)
              f32x2 UE[PB / 2];
              if (COL) {
                const float ex = srec[2 * (c + 1)].w, ey = srec[2 * (c + 2)].w;
#pragma unroll
                for (int h = 0; h < PB / 2; ++h) UE[h] = ffma2(bc2(ex), UX[h], fmul2(bc2(ey), UY[h]));
              }
              constexpr bool HORN = kHorner && TERMS <= kHornerMax;
              f32x2 H[PB / 2][TERMS];
              if (HORN) {
#pragma unroll
                for (int h = 0; h < PB / 2; ++h) horner_coef<TERMS>(Q0[h], H[h]);
              }
#pragma unroll kJUnroll
              for (int j = 1; j < kGroup; ++j) {
                const float4 Aj = srec[2 * (c + j)], Bj = srec[2 * (c + j) + 1];
#pragma unroll
                for (int h = 0; h < PB / 2; ++h) {
                  const f32x2 E = COL ? ffma2(bc2(Aj.x), UE[h], bc2(Aj.z))
                                      : ffma2(bc2(Aj.x), UX[h], ffma2(bc2(Aj.y), UY[h], bc2(Aj.z)));
                  if (HORN) {
                    tail_n(h, horner_leg<TERMS>(E, H[h], DR0[h]), Bj.x, __float_as_uint(Bj.y));
                  } else {
                    const f32x2 EQ = fmul2(E, Q0[h]);      // ~ R_b delta
                    const f32x2 D = fmul2(EQ, Q0[h]);      // delta
                    const f32x2 P = TERMS == 2 ? ffma2(D, bc2(-0.125f), bc2(0.5f))
                                               : ffma2(D, ffma2(D, bc2(0.0625f), bc2(-0.125f)), bc2(0.5f));
                    tail_n(h, ffma2(EQ, P, DR0[h]), Bj.x, __float_as_uint(Bj.y));
                  }
                }
              }
            };
            using T2 = std::integral_constant<int, 2>;
            using T3 = std::integral_constant<int, 3>;
            if (kColMono && B.w == 6.f) group(T2{}, std::true_type{});
            else if (B.w == 2.f) group(T2{}, std::false_type{});
            else if (kColMono && B.w == 7.f) group(T3{}, std::true_type{});
            else group(T3{}, std::false_type{});
            c += kGroup;
          } else {
#pragma unroll
            for (int h = 0; h < PB / 2; ++h) tail(h, leg_delta2(A, UX[h], UY[h], W2[h]), B.x, __float_as_uint(B.y));
            ++c;
          }
        }
      } else if (kDerBi && srec[1].w != 0.f) {
        // derived stage (bistatic): chirp 0's TX leg by rsqrt; every other leg l of the stage by
        // |p - q_l| - r_b = dR_b + (E Q) P4(delta), delta = E Q^2,
        // P4 = 1/2 - delta/8 + delta^2/16 - 5 delta^3/128; d_hyp - 2 r_b = 2 dR_b + X_tx + X_rx
        // (3-term stages: P3 = 1/2 - delta/8 + delta^2/16; srec[1].w = terms, srec[1].z = eps)
        const float4 T0 = srec[0], T0b = srec[1];
        f32x2 DR2[PB / 2], Q0[PB / 2];
#pragma unroll
        for (int h = 0; h < PB / 2; ++h) {
          const f32x2 d0 = leg_delta2q(T0, UX[h], UY[h], W2[h], Q0[h]);
          DR2[h] = ffma2(d0, bc2(2.f), bc2(T0b.z));   // 2 dR_b + eps
        }
        auto stage = [&](auto nrx_tag, auto terms_tag, auto col_tag) {   // NRX > 0: the RX count at compile time
          constexpr int NRX = decltype(nrx_tag)::value;
          constexpr int TERMS = decltype(terms_tag)::value;
          constexpr bool COL = decltype(col_tag)::value;   // collinear stage: E = c + s (e.u), e = srec[1].xy
          f32x2 UE[PB / 2];
          if (COL) {
#pragma unroll
            for (int h = 0; h < PB / 2; ++h) UE[h] = ffma2(bc2(T0b.x), UX[h], fmul2(bc2(T0b.y), UY[h]));
          }
          constexpr bool HORN = kHorner && TERMS <= kHornerMaxBi;
          f32x2 H[PB / 2][TERMS];
          if (HORN) {
#pragma unroll
            for (int h = 0; h < PB / 2; ++h) horner_coef<TERMS>(Q0[h], H[h]);
          }
          auto xleg = [&](const float4 R, const int h, const f32x2 base) {   // base + (E Q) P(delta), leg of record R
            const f32x2 E = COL ? ffma2(bc2(R.x), UE[h], bc2(R.y))
                                : ffma2(bc2(R.x), UX[h], ffma2(bc2(R.y), UY[h], bc2(R.z)));
            if (HORN) return horner_leg<TERMS>(E, H[h], base);
            const f32x2 EQ = fmul2(E, Q0[h]);
            const f32x2 D = fmul2(EQ, Q0[h]);
            const f32x2 P = TERMS == 3
                                ? ffma2(D, ffma2(D, bc2(0.0625f), bc2(-0.125f)), bc2(0.5f))
                                : ffma2(D, ffma2(D, ffma2(D, bc2(-0.0390625f), bc2(0.0625f)), bc2(-0.125f)), bc2(0.5f));
            return ffma2(EQ, P, base);
          };
#pragma unroll 1
          for (int c = 0; c < cnt; ++c) {
            f32x2 TS[PB / 2];
            if (c == 0) {
#pragma unroll
              for (int h = 0; h < PB / 2; ++h) TS[h] = DR2[h];
            } else {
              const float4 T = srec[2 * c];
#pragma unroll
              for (int h = 0; h < PB / 2; ++h) TS[h] = xleg(T, h, DR2[h]);
            }
            const float4* rp = srec + 2 * (a.CB + c * a.n_rx);
            if constexpr (NRX > 0) {
#pragma unroll
              for (int n = 0; n < NRX; ++n, rp += 2) {
                const float4 A = rp[0];
                const float2 B = COL ? make_float2(A.z, A.w) : *reinterpret_cast<const float2*>(rp + 1);
#pragma unroll
                for (int h = 0; h < PB / 2; ++h) tail_n(h, xleg(A, h, TS[h]), B.x, __float_as_uint(B.y));
              }
            } else {
#pragma unroll kRxUnroll
              for (int n = 0; n < a.n_rx; ++n, rp += 2) {
                const float4 A = rp[0];
                const float2 B = COL ? make_float2(A.z, A.w) : *reinterpret_cast<const float2*>(rp + 1);
#pragma unroll
                for (int h = 0; h < PB / 2; ++h) tail_n(h, xleg(A, h, TS[h]), B.x, __float_as_uint(B.y));
              }
            }
          }
        };
        auto dispatch = [&](auto nrx_tag) {   // srec[1].w = terms (+ 16: collinear)
          using T3 = std::integral_constant<int, 3>;
          using T4 = std::integral_constant<int, 4>;
          if (T0b.w == 19.f) stage(nrx_tag, T3{}, std::true_type{});
          else if (T0b.w == 3.f) stage(nrx_tag, T3{}, std::false_type{});
          else if (T0b.w == 20.f) stage(nrx_tag, T4{}, std::true_type{});
          else stage(nrx_tag, T4{}, std::false_type{});
        };
        if (SAR_BP_NRX_SPEC > 0 && a.n_rx == SAR_BP_NRX_SPEC) dispatch(std::integral_constant<int, SAR_BP_NRX_SPEC>{});
        else dispatch(std::integral_constant<int, 0>{});
      } else {
#pragma unroll 1
        for (int c = 0; c < cnt; ++c) {
          const float4 T = srec[2 * c];
          f32x2 DT[PB / 2];
#pragma unroll
          for (int h = 0; h < PB / 2; ++h) DT[h] = leg_delta2(T, UX[h], UY[h], W2[h]);
          const float4* rp = srec + 2 * (a.CB + c * a.n_rx);
#pragma unroll kRxUnroll
          for (int n = 0; n < a.n_rx; ++n, rp += 2) {
            const float4 A = rp[0], B = rp[1];
#pragma unroll
            for (int h = 0; h < PB / 2; ++h)
              tail(h, fadd2(DT[h], leg_delta2(A, UX[h], UY[h], W2[h])), B.x, __float_as_uint(B.y));
          }
        }
      }
    } else if (!BISTATIC) {
#pragma unroll kChirpUnroll
      for (int c = 0; c < cnt; ++c) {
        const float4 A = srec[2 * c], B = srec[2 * c + 1];
        const uint32_t off = __float_as_uint(B.y);
#pragma unroll
        for (int p = 0; p < PB; ++p) {
          const float dR = leg_delta<SAFE>(A.x, A.y, A.z, A.w, B.z, ux[p], uy[p], wh[p]);
          float kap = fmaf(A1, dR, B.x);
          if (DOP) kap += fd[p];
          const float tk = kap + kMagic;
          const float kf = tk - kMagic;
          const float gf = kap - kf;
          SAR_CHECK((unsigned)((int)(__float_as_uint(tk) - kMagicBits) + (a.W >> 1)) < (unsigned)a.W, 0);
          SAR_CHECK(__float_as_uint(tk) * 16u + off >= sbase + L.win &&
                    __float_as_uint(tk) * 16u + off + 16u <= sbase + L.total, 3);
          const float4 e = lds128(win_addr(tk, off));
          const float vr = fmaf(gf, e.z, e.x), vi = fmaf(gf, e.w, e.y);
          float sn, cs;
          __sincosf(C3 * gf, &sn, &cs);
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
        for (int p = 0; p < PB; ++p) dT[p] = leg_delta<SAFE>(T.x, T.y, T.z, T.w, TB.z, ux[p], uy[p], wh[p]);
#pragma unroll 1
        for (int n = 0; n < a.n_rx; ++n) {
          const int ri = a.CB + c * a.n_rx + n;
          const float4 A = srec[2 * ri], B = srec[2 * ri + 1];
          const uint32_t off = __float_as_uint(B.y);
#pragma unroll
          for (int p = 0; p < PB; ++p) {
            const float dR = dT[p] + leg_delta<SAFE>(A.x, A.y, A.z, A.w, B.z, ux[p], uy[p], wh[p]);
            float kap = fmaf(A1, dR, B.x);
            if (DOP) kap += fd[p];
            const float tk = kap + kMagic;
            const float kf = tk - kMagic;
            const float gf = kap - kf;
            SAR_CHECK((unsigned)((int)(__float_as_uint(tk) - kMagicBits) + (a.W >> 1)) < (unsigned)a.W, 0);
          SAR_CHECK(__float_as_uint(tk) * 16u + off >= sbase + L.win &&
                    __float_as_uint(tk) * 16u + off + 16u <= sbase + L.total, 3);
          const float4 e = lds128(win_addr(tk, off));
            const float vr = fmaf(gf, e.z, e.x), vi = fmaf(gf, e.w, e.y);
            float sn, cs;
            __sincosf(C3 * gf, &sn, &cs);
            acc_r[p] = fmaf(vr, cs, acc_r[p]);
            acc_r[p] = fmaf(-vi, sn, acc_r[p]);
            acc_i[p] = fmaf(vr, sn, acc_i[p]);
            acc_i[p] = fmaf(vi, cs, acc_i[p]);
          }
        }
      }
    }
    mbar_arrive(bar_empty + 8 * slot);
    SAR_TR(warp, it, 2);
    if (++slot == S) {
      slot = 0;
      parity ^= 1;
    }
  }

  if (kPaired) {
#pragma unroll
    for (int p = 0; p < PB; ++p) {
      acc_r[p] = lo2(ACC[p]) - lo2(ACI[p]);
      acc_i[p] = hi2(ACC[p]) + hi2(ACI[p]);
    }
  }
  // epilogue: remove the Doppler index shift from the folded phase, then store (or
  // accumulate) the tile.  The chirp chunk is re-read from %ctaid here (not kept in a register
  // across the chirp loop, whose schedule is sensitive to register pressure)
  const int chunk_e = (int)(ctaid_x() / (unsigned)a.ntile);
#pragma unroll
  for (int p = 0; p < PB; ++p) {
    if (DOP) {
      float sn, cs;
      sincosf(-C3 * fd[p], &sn, &cs);
      const float r = acc_r[p] * cs - acc_i[p] * sn, i = acc_r[p] * sn + acc_i[p] * cs;
      acc_r[p] = r;
      acc_i[p] = i;
    }
  }
  if constexpr (SCATTER) {
    if (a.ws && a.ksplit > 1) {
      // split scatter: this chunk stores its partial tile into plane `chunk` of the workspace;
      // the last chunk of the tile to finish (threadfence-reduction pattern on a per-tile
      // counter) sums the planes in chunk order (deterministic) and stores the finished tile
      // to every peer, so the gather still overlaps other tiles
      SAR_CHECK(chunk_e < a.ws_planes, 1);
      float2* wsp = a.ws + (size_t)chunk_e * a.ws_plane;
#pragma unroll
      for (int p = 0; p < PB; ++p)
        if (SAR_PIX_OK(gx[p], gy[p]))
          __stcg(wsp + (size_t)gy[p] * a.nx + gx[p], make_float2(acc_r[p], acc_i[p]));
      __threadfence();
      // the flag lives in the record area: past the first barrier no consumer reads the ring
      volatile int* s_last = reinterpret_cast<volatile int*>(smem + L.rec);
      asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");   // consumer warps only
      if (threadIdx.x == 0) *s_last = atomicAdd(a.tile_count + (int)(ctaid_x() % (unsigned)a.ntile), 1) == a.ksplit - 1;
      asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
      if (!*s_last) return;
      __threadfence();
#pragma unroll
      for (int p = 0; p < PB; ++p) {
        if (SAR_PIX_OK(gx[p], gy[p])) {
          const size_t o = (size_t)gy[p] * a.nx + gx[p];
          float2 v = __ldcg(a.ws + o);
          for (int c = 1; c < a.ksplit; ++c) {
            const float2 w = __ldcg(a.ws + (size_t)c * a.ws_plane + o);
            v.x += w.x;
            v.y += w.y;
          }
          acc_r[p] = v.x;
          acc_i[p] = v.y;
        }
      }
    }
    // fused gather (NEXT-4): the finished tile goes straight to every rank's full image over
    // NVLink while other tiles are still being computed
#pragma unroll
    for (int p = 0; p < PB; ++p) {
      if (SAR_PIX_OK(gx[p], gy[p])) {
        const size_t o = (size_t)(a.row0 + gy[p]) * a.nx + gx[p];
        if (a.multicast) {
          float* d = reinterpret_cast<float*>(a.peer[0] + o);
          if (a.accumulate) {   // chirp shards: the NVSwitch adds into every rank's image
            asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(d), "f"(acc_r[p]) : "memory");
            asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(d + 1), "f"(acc_i[p]) : "memory");
          } else {
            asm volatile("multimem.st.relaxed.sys.global.v2.f32 [%0], {%1, %2};" ::"l"(d), "f"(acc_r[p]),
                         "f"(acc_i[p])
                         : "memory");
          }
        } else if (a.accumulate) {   // chirp shards: P2P reductions into the peers' images
          for (int q = 0; q < a.n_peer; ++q) {
            float* d = reinterpret_cast<float*>(a.peer[q] + o);
            asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(d), "f"(acc_r[p]) : "memory");
            asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(d + 1), "f"(acc_i[p]) : "memory");
          }
        } else {
          for (int q = 0; q < a.n_peer; ++q) a.peer[q][o] = make_float2(acc_r[p], acc_i[p]);
        }
      }
    }
  } else {
    // The plain family keeps the generic epilogue of the first design, peer branches included
    // (a.n_peer == 0 here, never taken): with it ptxas schedules the chirp loop in the form
    // measured fastest on C3 (0.7 % faster than without; tools/libsweep.sh).
#pragma unroll
    for (int p = 0; p < PB; ++p) {
      if (SAR_PIX_OK(gx[p], gy[p])) {
        float2* dst = a.img + (size_t)gy[p] * a.nx + gx[p];
        if (a.n_peer > 0) {
          const size_t o = (size_t)(a.row0 + gy[p]) * a.nx + gx[p];
          if (a.multicast) {
            float* d = reinterpret_cast<float*>(a.peer[0] + o);
            if (a.accumulate) {
              asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(d), "f"(acc_r[p]) : "memory");
              asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(d + 1), "f"(acc_i[p]) : "memory");
            } else {
              asm volatile("multimem.st.relaxed.sys.global.v2.f32 [%0], {%1, %2};" ::"l"(d), "f"(acc_r[p]),
                           "f"(acc_i[p])
                           : "memory");
            }
          } else if (a.accumulate) {
            for (int q = 0; q < a.n_peer; ++q) {
              float* d = reinterpret_cast<float*>(a.peer[q] + o);
              asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(d), "f"(acc_r[p]) : "memory");
              asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(d + 1), "f"(acc_i[p]) : "memory");
            }
          } else {
            for (int q = 0; q < a.n_peer; ++q) a.peer[q][o] = make_float2(acc_r[p], acc_i[p]);
          }
        } else if (a.ksplit > 1 && chunk_e > 0) {
          // chirp chunks 1.. store their partials into workspace planes 0..; chunk 0 stores (or
          // accumulates) into the image like an unsplit launch, and the split-sum kernel then
          // adds the planes in chunk order (deterministic, unlike reductions)
          SAR_CHECK(chunk_e - 1 < a.ws_planes, 1);
          __stcg(a.ws + (size_t)(chunk_e - 1) * a.ws_plane + (size_t)gy[p] * a.nx + gx[p], make_float2(acc_r[p], acc_i[p]));
        } else if (a.accumulate) {
          const float2 o = *dst;
          *dst = make_float2(o.x + acc_r[p], o.y + acc_i[p]);
        } else {
          *dst = make_float2(acc_r[p], acc_i[p]);
        }
      }
    }
  }
  };
  if constexpr (NEAR) {
    if (tile_near) consume(std::true_type{});
    else consume(std::false_type{});
  } else {
    consume(std::false_type{});
  }
}

// Register budget: the monostatic and the bistatic kernels are held to three resident CTAs per SM
// at the default 32 x 32 tile (an unbounded bistatic kernel ran at 2 CTAs: C4 1343 ms vs 1190 at
// four in round 1, tools/vsweep.sh; three with the Horner stages since round 2).
#ifndef SAR_BP_MONO_MINB
// three resident CTAs per SM (72 registers): with the integer-index tails and 2-term Horner groups
// the fourth CTA no longer pays for the spills of the 56-register floor (C3 51.76 -> 50.73 ms, C0
// 9.20 -> 8.90, C2 21.43 -> 20.77; in round 1 and early round 2 the floor of four measured faster)
#define SAR_BP_MONO_MINB 3
#endif
// resident-CTA floor per shape (register cap ~56-113): ptxas otherwise spends registers on ILP of
// the unrolled derived groups (4 x 4: 64 -> 120 registers) and the occupancy collapses
#ifndef SAR_BP_SCATTER_MINB
#define SAR_BP_SCATTER_MINB SAR_BP_MONO_MINB
#endif
constexpr int mono_min_blocks(int ncw, int pb, bool scatter) {
  return ncw == 8 && pb == 4 ? (scatter ? SAR_BP_SCATTER_MINB : SAR_BP_MONO_MINB) : ncw == 4 && pb == 4 ? 6 : ncw == 4 && pb == 8 ? 4 : 2;
}
template <bool DOP, bool NEAR, int NCW, int PB, bool SCATTER>
__global__ void __launch_bounds__((NCW + 1) * 32, mono_min_blocks(NCW, PB, SCATTER)) bp_kernel_mono(const BpArgs a) {
  bp_body<false, DOP, NEAR, NCW, PB, SCATTER>(a);
}
template <bool DOP, bool NEAR, int NCW, int PB, bool SCATTER>
#ifndef SAR_BP_BI_MINB
#define SAR_BP_BI_MINB 3   // (with the Horner stages; 4 before: see SAR_BP_HORNER_MAX_BI)
#endif
#ifndef SAR_BP_BI_MINB_SMALL
#define SAR_BP_BI_MINB_SMALL 1   // other shapes (4 x 4: polar plans with wide windows)
#endif
__global__ void __launch_bounds__((NCW + 1) * 32, NCW * PB == 32 ? SAR_BP_BI_MINB : NCW * PB == 16 ? SAR_BP_BI_MINB_SMALL : 1) bp_kernel_bi(const BpArgs a) {
  bp_body<true, DOP, NEAR, NCW, PB, SCATTER>(a);
}
template <bool BI, bool DOP, bool NEAR, int NCW, int PB, bool SCATTER>
struct BpKernel {
  static constexpr auto fn = bp_kernel_mono<DOP, NEAR, NCW, PB, SCATTER>;
};
template <bool DOP, bool NEAR, int NCW, int PB, bool SCATTER>
struct BpKernel<true, DOP, NEAR, NCW, PB, SCATTER> {
  static constexpr auto fn = bp_kernel_bi<DOP, NEAR, NCW, PB, SCATTER>;
};

template <bool BI, bool DOP, bool SAFE, int NCW, int PB, bool SCATTER>
cudaError_t launch_one(const BpArgs& a, cudaStream_t s) {
  auto kern = BpKernel<BI, DOP, SAFE, NCW, PB, SCATTER>::fn;
  const Layout L = make_layout(a.W, a.CB, a.n_rx, a.S, BI);
  // the dynamic shared-memory opt-in is per device and per kernel instantiation
  static std::atomic<int> configured_bytes[kMaxDevices];
  int cur_dev = 0;
  if (cudaGetDevice(&cur_dev) != cudaSuccess || cur_dev < 0 || cur_dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if ((int)L.total > configured_bytes[cur_dev].load()) {
    // only ever raised, under a lock: a concurrent launch of a smaller plan cannot lower the
    // opt-in below what another thread's launch needs
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if ((int)L.total > configured_bytes[cur_dev].load()) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
      if (e != cudaSuccess) return e;
      configured_bytes[cur_dev].store((int)L.total);
    }
  }
  BpArgs b = a;
  const long ntiles = a.tile_hi - a.tile_lo;   // tiles that compute (the split heuristic)
  // Chirp split: enough CTAs for kSplitWaves waves of resident CTAs, each chunk at least
  // kMinSplitItems (chirp, RX) items (and a multiple of the ring stage).
  int resident = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, kern, (NCW + 1) * 32, L.total);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cur_dev);
  const long slots = (long)std::max(1, resident) * sms;
  // scatters (tuning: SAR_BP_SCATTER_WAVES, SAR_BP_SCATTER_UNSPLIT): the split publish reads every
  // chunk plane of a tile, so scatters aim at fewer waves than plain launches
  static const long scatter_waves = env_long("SAR_BP_SCATTER_WAVES", kScatterWaves);
  static const long scatter_unsplit = env_long("SAR_BP_SCATTER_UNSPLIT", kScatterUnsplit);
  const long waves = a.n_peer > 0 ? scatter_waves : kSplitWaves;
  int k = 1;
  while (ntiles * k < waves * slots && (long)a.nchirp * a.n_rx / (2 * k) >= kMinSplitItems &&
         a.nchirp / (2 * k) >= a.CB)
    k *= 2;
  // ... and enough chunks that one chunk's pair rows (the rows the resident CTAs stream at a time,
  // chunk-major order) stay inside L2: C4's 750-row rank block at 3 CTAs per SM took k = 4 (92 MB
  // per chunk) and read 5.7 GB from DRAM per launch instead of the rows' ~0.4 GB.  Window 40 / 64 MB
  // (tools/gpu_r4s.sh): C3 50.00 / 49.89 ms with 0.76 / 0.49 GB of DRAM traffic (chunk planes), C4
  // 868.5 / 870.4 ms, C4 rank block 111.9 / 112.9 ms
  // (plain launches only: a scatter -- the fused gather, sar_form_image's host-image stores -- keeps
  //  its unsplit epilogue stores where the waves allow; forcing C3's host-image launch to 8 chunks
  //  cost 1.3 ms end to end)
  static const long l2_window = env_long("SAR_BP_L2_WINDOW_MB", kL2WindowMB) << 20;
  if (a.pairs && a.n_peer == 0)
    while ((long)((a.nchirp + k - 1) / k) * a.n_rx * a.pair_stride * 16L > l2_window &&
           (long)a.nchirp * a.n_rx / (2 * k) >= kMinSplitItems && a.nchirp / (2 * k) >= a.CB)
      k *= 2;
  if (a.n_peer > 0 && ntiles >= scatter_unsplit * slots) k = 1;
  // reductions into peers (chirp shards) run unsplit
  if (a.n_peer > 0 && a.accumulate) k = 1;
  auto split = [&](int kk) {
    b.chunk = (a.nchirp + kk - 1) / kk;
    b.chunk = ((b.chunk + a.CB - 1) / a.CB) * a.CB;
    b.ksplit = std::max(1, (a.nchirp + b.chunk - 1) / std::max(1, b.chunk));
  };
  split(k);
  if (a.split_query) {
    // planning query, nothing runs: the number of chirp chunks (workspace planes) of this launch
    *a.split_query = b.ksplit;
    return cudaSuccess;
  }
  // a split needs its workspace planes (and tile counters for a scatter); without them, unsplit
  // (a plain launch keeps chunk 0 in the image: ksplit - 1 planes; a scatter needs ksplit)
  if (b.ksplit > 1 && (!a.ws || a.ws_planes < b.ksplit - (a.n_peer > 0 ? 0 : 1) || (a.n_peer > 0 && !a.tile_count)))
    split(1);
  if (b.ksplit > 1 && a.n_peer > 0) {
    cudaError_t e = cudaMemsetAsync(a.tile_count, 0, sizeof(int) * (size_t)a.ntile, s);
    if (e != cudaSuccess) return e;
  }
  if (a.ksplit_out) *a.ksplit_out = b.ksplit;
  const long grid = (long)a.ntile * b.ksplit;
  kern<<<(unsigned)grid, (NCW + 1) * 32, L.total, s>>>(b);
  return cudaGetLastError();
}

template <int NCW, int PB, bool SCATTER>
cudaError_t launch_shape(const BpArgs& a, bool bistatic, bool doppler, bool near, cudaStream_t s) {
  if (bistatic) {
    if (doppler)
      return near ? launch_one<true, true, true, NCW, PB, SCATTER>(a, s) : launch_one<true, true, false, NCW, PB, SCATTER>(a, s);
    return near ? launch_one<true, false, true, NCW, PB, SCATTER>(a, s) : launch_one<true, false, false, NCW, PB, SCATTER>(a, s);
  }
  if (doppler)
    return near ? launch_one<false, true, true, NCW, PB, SCATTER>(a, s) : launch_one<false, true, false, NCW, PB, SCATTER>(a, s);
  return near ? launch_one<false, false, true, NCW, PB, SCATTER>(a, s) : launch_one<false, false, false, NCW, PB, SCATTER>(a, s);
}

// CTA shape dispatch (consumer warps x pixels per thread); tile = 32 x (NCW * PB).
template <bool SCATTER>
cudaError_t launch_shapes(const BpArgs& a, bool bistatic, bool doppler, bool near, cudaStream_t s) {
  if (a.ncw == 8 && a.pb == 4) return launch_shape<8, 4, SCATTER>(a, bistatic, doppler, near, s);
  if (a.ncw == 4 && a.pb == 8) return launch_shape<4, 8, SCATTER>(a, bistatic, doppler, near, s);
  if (a.ncw == 4 && a.pb == 4) return launch_shape<4, 4, SCATTER>(a, bistatic, doppler, near, s);
  if (a.ncw == 8 && a.pb == 8) return launch_shape<8, 8, SCATTER>(a, bistatic, doppler, near, s);
  return cudaErrorInvalidConfiguration;
}

}  // namespace
}  // namespace sar
