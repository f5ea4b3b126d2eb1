// libsar C ABI: plan maths, validation, constant tables, launches (include/sar_bp.h).
//
// Citations: P:Lnnn = PAPER.md line (arXiv 2306.09784); A1..A17 = readings in DESIGN.md.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <string>
#include <vector>

#include "sar_internal.h"

namespace {

thread_local std::string g_last_error;

sar_status_t fail(sar_status_t st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

sar_status_t cuda_fail(cudaError_t e, const char* what) {
  return fail(SAR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

bool finite_pos(double v) { return isfinite(v) && v > 0.0; }

// Minimum and maximum Euclidean distance between two axis-aligned boxes.
void box_distance(const double alo[3], const double ahi[3], const double blo[3],
                  const double bhi[3], double* dmin, double* dmax) {
  double s_min = 0.0, s_max = 0.0;
  for (int k = 0; k < 3; ++k) {
    const double gap = std::max(0.0, std::max(alo[k] - bhi[k], blo[k] - ahi[k]));
    const double far = std::max(fabs(ahi[k] - blo[k]), fabs(bhi[k] - alo[k]));
    s_min += gap * gap;
    s_max += far * far;
  }
  *dmin = sqrt(s_min);
  *dmax = sqrt(s_max);
}

struct Derived {
  sar_plan_info_t info;
  double rho;       // tile half-diagonal, max over tiles (near-field test)
  double win_rho;   // per-leg half spread of |p - q| over a tile, max over tiles (window)
  bool near_field;
  int ncw, pb, stages;
};

// Polar grid (Measure E) -> bounding box of the annular sector and a Cartesian stand-in
// (nx = n_th, ny = n_r) for the row/column bookkeeping shared with Cartesian plans.
sar_status_t polar_box(const sar_polar_grid_t* pg, double lo[3], double hi[3], sar_grid_t* stand_in) {
  if (!pg) return fail(SAR_ERR_INVALID_ARGUMENT, "null polar grid");
  if (!finite_pos(pg->dr) || !finite_pos(pg->dth) || !(pg->r0 >= 0.0) || !isfinite(pg->r0) ||
      !isfinite(pg->th0) || !isfinite(pg->xc) || !isfinite(pg->yc) || !isfinite(pg->zc) || pg->n_th < 1 ||
      pg->n_r < 1)
    return fail(SAR_ERR_INVALID_ARGUMENT, "polar grid needs r0 >= 0, dr, dth > 0, n_th, n_r >= 1");
  const double th1 = pg->th0 + (pg->n_th - 1) * pg->dth;
  if (th1 - pg->th0 >= 2.0 * sar::kPi) return fail(SAR_ERR_INVALID_ARGUMENT, "polar grid spans >= 2 pi");
  const double r1 = pg->r0 + (pg->n_r - 1) * pg->dr;
  lo[0] = lo[1] = 1e300;
  hi[0] = hi[1] = -1e300;
  auto add = [&](double rr, double th) {
    const double x = pg->xc + rr * sin(th), y = pg->yc + rr * cos(th);
    lo[0] = std::min(lo[0], x); hi[0] = std::max(hi[0], x);
    lo[1] = std::min(lo[1], y); hi[1] = std::max(hi[1], y);
  };
  for (double rr : {pg->r0, r1}) {
    add(rr, pg->th0);
    add(rr, th1);
    const int k0 = (int)floor(pg->th0 / (0.5 * sar::kPi)), k1 = (int)ceil(th1 / (0.5 * sar::kPi));
    for (int k = k0; k <= k1; ++k) {  // bearings where sin or cos is extreme
      const double t = k * 0.5 * sar::kPi;
      if (t > pg->th0 && t < th1) add(rr, t);
    }
  }
  lo[2] = hi[2] = pg->zc;
  *stand_in = sar_grid_t{pg->xc, pg->yc, pg->zc, pg->dr, pg->dr, pg->n_th, pg->n_r};
  return SAR_OK;
}

// Crop of the one-sided spectrum a (sub-)grid needs: every two-way path from the declared
// antenna box to the grid's box (and, for a polar grid, through its centre) lies in
// [d_min, d_max]; bins [k_lo, k_hi] with interpolation margin, even row length.
sar_status_t crop_bins(const sar_radar_params_t* r, const sar_grid_t* g, const sar_box_t* b,
                       const sar_polar_grid_t* pg, double a1, double* d_min, double* d_max, long* k_lo,
                       long* k_hi) {
  double glo[3] = {g->x0, g->y0, g->z0};
  double ghi[3] = {g->x0 + (g->nx - 1) * g->dx, g->y0 + (g->ny - 1) * g->dy, g->z0};
  if (pg) {
    sar_grid_t tmp;
    sar_status_t st = polar_box(pg, glo, ghi, &tmp);
    if (st != SAR_OK) return st;
  }
  double dist_min, dist_max;
  box_distance(glo, ghi, b->lo, b->hi, &dist_min, &dist_max);
  if (pg) {
    // an annular sector is poorly described by its bounding box: also bound each leg
    // through the polar centre c, r - |q - c| <= |p - q| <= r + |q - c|
    double sc = 0.0;
    for (int cx = 0; cx < 2; ++cx)
      for (int cy = 0; cy < 2; ++cy)
        for (int cz = 0; cz < 2; ++cz) {
          const double ex = (cx ? b->hi[0] : b->lo[0]) - pg->xc, ey = (cy ? b->hi[1] : b->lo[1]) - pg->yc,
                       ez = (cz ? b->hi[2] : b->lo[2]) - pg->zc;
          sc = std::max(sc, sqrt(ex * ex + ey * ey + ez * ez));
        }
    const double r1 = pg->r0 + (pg->n_r - 1) * pg->dr;
    dist_min = std::max(dist_min, pg->r0 - sc);
    dist_max = std::min(dist_max, r1 + sc);
  }
  *d_min = 2.0 * dist_min;  // each leg lies in [dist_min, dist_max]
  *d_max = 2.0 * dist_max;
  const double dop = r->doppler_max_bins;
  const long half = r->fft_len / 2;
  long lo_ = (long)floor(a1 * *d_min - dop) - 2;
  long hi_ = (long)floor(a1 * *d_max + dop) + 3;
  lo_ = std::max(0L, std::min(lo_, half));
  hi_ = std::max(lo_, std::min(hi_, half));
  // even row length (16-B aligned rows); the extra bin may be N/2 + 1, which the range
  // compression writes as 0 (A8)
  if ((hi_ - lo_ + 1) & 1) ++hi_;
  *k_lo = lo_;
  *k_hi = hi_;
  return SAR_OK;
}

// Host-side plan maths shared by sar_plan_geometry and sar_plan_create (pg: polar grid or
// nullptr; g then is the Cartesian stand-in from polar_box).
sar_status_t derive(const sar_radar_params_t* r, const sar_grid_t* g, const sar_box_t* b,
                    Derived* out, const sar_polar_grid_t* pg = nullptr) {
  if (!r || !g || !b || !out) return fail(SAR_ERR_INVALID_ARGUMENT, "null argument");
  if (!finite_pos(r->f0_hz) || !finite_pos(r->bandwidth_hz) || !finite_pos(r->chirp_s) ||
      !finite_pos(r->pri_s) || !finite_pos(r->sample_rate_hz))
    return fail(SAR_ERR_INVALID_ARGUMENT, "radar times and frequencies must be finite and > 0");
  if (r->pri_s < r->chirp_s) return fail(SAR_ERR_INVALID_ARGUMENT, "pri_s must be >= chirp_s");
  if (r->n_samples < 2) return fail(SAR_ERR_INVALID_ARGUMENT, "n_samples must be >= 2");
  if (llround(r->sample_rate_hz * r->chirp_s) != r->n_samples)
    return fail(SAR_ERR_INVALID_ARGUMENT, "round(sample_rate_hz * chirp_s) must equal n_samples");
  if (r->fft_len < r->n_samples || r->fft_len > 16384 || (r->fft_len & (r->fft_len - 1)))
    return fail(SAR_ERR_INVALID_ARGUMENT, "fft_len must be a power of two in [n_samples, 16384]");
  if (r->n_chirps < 1 || r->n_rx < 1)
    return fail(SAR_ERR_INVALID_ARGUMENT, "n_chirps and n_rx must be >= 1");
  if (r->range_window != 0 && r->range_window != 1)
    return fail(SAR_ERR_INVALID_ARGUMENT, "range_window must be 0 (rect) or 1 (Hann)");
  if (!(r->doppler_max_bins >= 0.0f) || !isfinite(r->doppler_max_bins))
    return fail(SAR_ERR_INVALID_ARGUMENT, "doppler_max_bins must be finite and >= 0");
  if (!finite_pos(g->dx) || !finite_pos(g->dy) || !isfinite(g->x0) || !isfinite(g->y0) ||
      !isfinite(g->z0) || g->nx < 1 || g->ny < 1)
    return fail(SAR_ERR_INVALID_ARGUMENT, "grid needs finite origin, dx, dy > 0, nx, ny >= 1");
  for (int k = 0; k < 3; ++k)
    if (!isfinite(b->lo[k]) || !isfinite(b->hi[k]) || b->lo[k] > b->hi[k])
      return fail(SAR_ERR_INVALID_ARGUMENT, "antenna box needs finite lo <= hi");

  sar_plan_info_t& I = out->info;
  memset(&I, 0, sizeof(I));
  const double N = (double)r->fft_len;
  I.chirp_rate_hz_per_s = r->bandwidth_hz / r->chirp_s;                    // mu
  I.a1_bins_per_m = I.chirp_rate_hz_per_s * N / (sar::kLightSpeed * r->sample_rate_hz);
  I.c2_cycles_per_m = r->f0_hz / sar::kLightSpeed;                         // f0 / c (A3)

  long k_lo, k_hi;
  sar_status_t cst = crop_bins(r, g, b, pg, I.a1_bins_per_m, &I.d_min_m, &I.d_max_m, &k_lo, &k_hi);
  if (cst != SAR_OK) return cst;
  const double dop = r->doppler_max_bins;
  const double dist_min = 0.5 * I.d_min_m;   // one leg
  I.k_lo = (int32_t)k_lo;
  I.n_bins = (int32_t)(k_hi - k_lo + 1);

  // BP CTA shape and shared-memory ring (tuning override: SAR_BP_SHAPE="ncw,pb,stages,cb")
  int ncw = 8, pb = 4, stages = 0, cb = 0;
  bool shape_env = false;
  if (const char* env = getenv("SAR_BP_SHAPE")) {
    int v[4] = {0, 0, 0, 0};
    if (sscanf(env, "%d,%d,%d,%d", &v[0], &v[1], &v[2], &v[3]) >= 2 && sar::bp_shape_supported(v[0], v[1])) {
      ncw = v[0];
      pb = v[1];
      stages = v[2];
      cb = v[3];
      shape_env = true;
    }
  }
  // Tile geometry of a CTA shape; polar grids whose 32 x 32 tiles span a wide range window
  // (coarse range spacing, Measure E) take 32 x 16 tiles (C6p: 2.41 -> 2.22 ms).
  for (int pass = 0;; ++pass) {
    out->ncw = ncw;
    out->pb = pb;
    I.tile_x = sar::kTileX;
    I.tile_y = ncw * pb;  // 32-pixel-wide rows of 8x4 patches: tile area = 32 * ncw * pb
    if (!pg) {
      const double hx = 0.5 * (I.tile_x - 1) * g->dx, hy = 0.5 * (I.tile_y - 1) * g->dy;
      out->rho = sqrt(hx * hx + hy * hy) * (1.0 + 1e-9) + 1e-12;
      out->win_rho = out->rho;   // triangle inequality: ||p - q| - |P_T - q|| <= |p - P_T|
    } else {
      // Per tile row (anchor radius rc, half extents hr in range and ht in bearing):
      //  * rho_T: farthest tile corner from the anchor (the annular patch lies within it);
      //  * window: the triangle bound rho_T is loose for polar tiles seen from near the polar
      //    centre c.  With s = q - c (horizontal part s_h), |d|p - q|/dr| <= 1 and
      //    |d|p - q|/dth| = r |s_h . e_perp| / |p - q| <= r s_h / (r - s_h), so moving from the
      //    anchor first in range, then in bearing at radius r >= r_in = rc - hr gives
      //    ||p - q| - |P_T - q|| <= hr + ht r_in s_h / (r_in - s_h) when r_in > s_h.
      const double ht = 0.5 * (I.tile_x - 1) * pg->dth, hr = 0.5 * (I.tile_y - 1) * pg->dr;
      const int tiles_r = (pg->n_r + I.tile_y - 1) / I.tile_y;
      double sh = 0.0;
      for (int cx = 0; cx < 2; ++cx)
        for (int cy = 0; cy < 2; ++cy)
          sh = std::max(sh, hypot((cx ? b->hi[0] : b->lo[0]) - pg->xc, (cy ? b->hi[1] : b->lo[1]) - pg->yc));
      double rho = 0.0, wrho = 0.0;
      for (int t = 0; t < tiles_r; ++t) {
        const double rc = pg->r0 + (t * I.tile_y + 0.5 * (I.tile_y - 1)) * pg->dr;
        double rho_t = 0.0;
        for (int sr = -1; sr <= 1; sr += 2)
          for (int st2 = -1; st2 <= 1; st2 += 2) {
            const double rr = rc + sr * hr, dt = st2 * ht;
            const double dx = rr * sin(dt), dy = rr * cos(dt) - rc;
            rho_t = std::max(rho_t, sqrt(dx * dx + dy * dy));
          }
        double w_t = rho_t;
        const double r_in = rc - hr;
        if (r_in > sh * (1.0 + 1e-9)) w_t = std::min(w_t, hr + ht * r_in * sh / (r_in - sh));
        rho = std::max(rho, rho_t);
        wrho = std::max(wrho, w_t);
      }
      out->rho = rho * (1.0 + 1e-6) + 1e-9;
      out->win_rho = wrho * (1.0 + 1e-6) + 1e-9;
    }
    const double w_try = ceil(2.0 * (2.0 * I.a1_bins_per_m * out->win_rho + dop)) + 4.0;
    if (pass == 0 && pg && !shape_env && w_try > 80.0) {
      ncw = 4;
      pb = 4;
      continue;
    }
    break;
  }
  const double kap_half = 2.0 * I.a1_bins_per_m * out->win_rho + dop;
  const double w = ceil(2.0 * kap_half) + 4.0;
  if (w > 4096.0)
    return fail(SAR_ERR_INVALID_ARGUMENT,
                "pixel spacing too coarse: one BP tile spans more than 4096 range bins");
  I.window_bins = (int32_t)w;
  I.window_half_bins = kap_half;
  I.tile_rho_m = out->rho;
  const bool bistatic = r->n_rx > 1;
  const bool auto_cb = cb <= 0, auto_stages = stages <= 0;
  auto smem = [&](int cb_, int st) {
    return sar::bp_smem_bytes(I.window_bins, cb_, r->n_rx, st, bistatic);
  };
  // ring budget per CTA: the monostatic kernel keeps three CTAs per SM resident (72 registers),
  // so up to ~64 KB each; wide windows take fewer chirps per stage (in steps of the derived-chirp
  // group while possible).  Measured (tools/gpu_r4e.sh): C0 (W = 59) 32 chirps x 2 stages 8.85 ms vs
  // 24: 8.93, 16: 9.16; C3 (W = 26) 4 stages of 32: 50.31 ms vs 3: 50.73, 2: 51.42
  const size_t ring_budget = bistatic ? 48 * 1024 : 64 * 1024;
  if (auto_cb && !bistatic) {
    cb = 32;
    while (cb > 1 && smem(cb, 2) > 64 * 1024) cb = cb > 8 ? cb - 8 : cb / 2;
  } else if (auto_cb) {
    // bistatic: long stages (~64 (chirp, RX) items) amortise the stage's base leg and records over
    // more legs; the largest count whose 2-stage ring fits in 64 KB.  Measured (tools/gpu_r3j.sh,
    // r4k.sh): C4 rank shard cb 8 -> 24: 121.0 -> 118.8 ms at four CTAs per SM; at three with Horner
    // stages cb 16 / 20 / 24 / 32: 114.1 / 116.0 / 115.6 / 117.2 ms (shorter stages keep more of them
    // within 3 series terms); C6 (W = 59) cb 2 -> 4: 11.36 -> 10.41 ms, cb 6 / 8: 11.45 / 16.9 ms
    cb = std::max(1, 64 / r->n_rx);
    while (cb > 1 && smem(cb, 2) > 64 * 1024) --cb;
  }
  for (;;) {
    const size_t stage_bytes = smem(cb, 2) - smem(cb, 1);
    int st = stages;
    // ring depth: as many stages as fit in the budget
    if (auto_stages) st = (int)std::min<size_t>(sar::kBpMaxStages, ring_budget / std::max<size_t>(1, stage_bytes));
    st = std::max(2, std::min(sar::kBpMaxStages, st));
    if (smem(cb, st) <= 200 * 1024) {
      stages = st;
      break;
    }
    if (!auto_cb || cb == 1)
      return fail(SAR_ERR_INVALID_ARGUMENT, "BP shared-memory ring does not fit (window too wide)");
    cb = std::max(1, cb / 2);
  }
  I.chirps_per_stage = cb;
  out->stages = stages;
  if ((int64_t)r->n_chirps * r->n_rx * (I.n_bins + 1) >= (int64_t)1 << 31)
    return fail(SAR_ERR_INVALID_ARGUMENT, "n_chirps * n_rx * n_bins must stay below 2^31");
  I.updates_per_image = (int64_t)g->nx * g->ny * r->n_chirps * r->n_rx;
  out->near_field = dist_min < 2.0 * out->rho + 1e-3;
  return SAR_OK;
}

template <class T>
sar_status_t dev_alloc(T** p, size_t count) {
  cudaError_t e = cudaMalloc((void**)p, std::max<size_t>(1, count) * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(SAR_ERR_NO_MEMORY, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  return SAR_OK;
}

struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess) ok = true;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

void free_plan(sar_plan_s* p) {
  if (!p) return;
  cudaFree(p->d_window);
  cudaFree(p->d_twiddle);
  cudaFree(p->d_rc_coef);
  cudaFree(p->d_rc_stw);
  cudaFree(p->d_ramp);
  cudaFree(p->d_binphase);

  cudaFree(p->w_raw);
  cudaFree(p->w_wsar);
  cudaFree(p->w_tx);
  cudaFree(p->w_rx);
  cudaFree(p->w_dop);
  cudaFree(p->w_prof);
  cudaFree(p->w_img);
  for (cudaEvent_t ev : p->w_ev)
    if (ev) cudaEventDestroy(ev);
  if (p->w_copy) cudaStreamDestroy(p->w_copy);
  delete p;
}

}  // namespace

extern "C" {

const char* sar_last_error(void) { return g_last_error.c_str(); }

const char* sar_version(void) { return "libsar 0.1 (sm_100a)"; }

sar_status_t sar_plan_geometry(const sar_radar_params_t* radar, const sar_grid_t* grid,
                               const sar_box_t* antenna_box, sar_plan_info_t* info) {
  if (!info) return fail(SAR_ERR_INVALID_ARGUMENT, "info is null");
  Derived d;
  sar_status_t st = derive(radar, grid, antenna_box, &d);
  if (st != SAR_OK) return st;
  *info = d.info;
  return SAR_OK;
}

sar_status_t sar_plan_geometry_polar(const sar_radar_params_t* radar, const sar_polar_grid_t* grid,
                                     const sar_box_t* antenna_box, sar_plan_info_t* info) {
  if (!info) return fail(SAR_ERR_INVALID_ARGUMENT, "info is null");
  sar_grid_t stand_in;
  double lo[3], hi[3];
  sar_status_t st = polar_box(grid, lo, hi, &stand_in);
  if (st != SAR_OK) return st;
  Derived d;
  st = derive(radar, &stand_in, antenna_box, &d, grid);
  if (st != SAR_OK) return st;
  *info = d.info;
  return SAR_OK;
}

static sar_status_t create_impl(const sar_radar_params_t* radar, const sar_grid_t* grid,
                                const sar_box_t* antenna_box, int32_t device, sar_plan_t* out,
                                const sar_polar_grid_t* pg);

sar_status_t sar_plan_create(const sar_radar_params_t* radar, const sar_grid_t* grid,
                             const sar_box_t* antenna_box, int32_t device, sar_plan_t* out) {
  return create_impl(radar, grid, antenna_box, device, out, nullptr);
}

sar_status_t sar_plan_create_polar(const sar_radar_params_t* radar, const sar_polar_grid_t* grid,
                                   const sar_box_t* antenna_box, int32_t device, sar_plan_t* out) {
  if (!out) return fail(SAR_ERR_INVALID_ARGUMENT, "out is null");
  *out = nullptr;
  sar_grid_t stand_in;
  double lo[3], hi[3];
  sar_status_t st = polar_box(grid, lo, hi, &stand_in);
  if (st != SAR_OK) return st;
  return create_impl(radar, &stand_in, antenna_box, device, out, grid);
}

static sar_status_t create_impl(const sar_radar_params_t* radar, const sar_grid_t* grid,
                                const sar_box_t* antenna_box, int32_t device, sar_plan_t* out,
                                const sar_polar_grid_t* pg) {
  if (!out) return fail(SAR_ERR_INVALID_ARGUMENT, "out is null");
  *out = nullptr;
  Derived d;
  sar_status_t st = derive(radar, grid, antenna_box, &d, pg);
  if (st != SAR_OK) return st;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return fail(SAR_ERR_UNSUPPORTED_DEVICE, "no such CUDA device");
  }
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess)
    return cuda_fail(e, "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(SAR_ERR_UNSUPPORTED_DEVICE,
                std::string("libsar is built for sm_100a only; device is ") + prop.name);
  DeviceGuard guard(device);
  if (!guard.ok) return cuda_fail(cudaGetLastError(), "cudaSetDevice");

  sar_plan_s* p = new (std::nothrow) sar_plan_s();
  if (!p) return fail(SAR_ERR_NO_MEMORY, "host allocation failed");
  p->radar = *radar;
  p->grid = *grid;
  p->polar = pg != nullptr;
  if (pg) p->pgrid = *pg;
  p->box = *antenna_box;
  p->info = d.info;
  p->device = device;
  p->near_field = d.near_field;
  p->tile_rho = d.rho;
  p->win_rho = d.win_rho;
  p->bp_ncw = d.ncw;
  p->bp_pb = d.pb;
  p->bp_stages = d.stages;
  {
    // per-device pool for the per-call pair-format rows: stream-ordered allocations that stay
    // warm across calls and plans (C5's frame plans share it); created once, never released
    static std::mutex pool_mutex;
    static cudaMemPool_t pools[sar::kMaxDevices] = {};
    std::lock_guard<std::mutex> lock(pool_mutex);
    if (device >= sar::kMaxDevices) {
      free_plan(p);
      return fail(SAR_ERR_UNSUPPORTED_DEVICE, "device index too large");
    }
    if (!pools[device]) {
      cudaMemPoolProps pp{};
      pp.allocType = cudaMemAllocationTypePinned;
      pp.handleTypes = cudaMemHandleTypeNone;
      pp.location.type = cudaMemLocationTypeDevice;
      pp.location.id = device;
      cudaError_t e = cudaMemPoolCreate(&pools[device], &pp);
      if (e != cudaSuccess) {
        pools[device] = nullptr;
        free_plan(p);
        return cuda_fail(e, "cudaMemPoolCreate");
      }
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    p->pool = pools[device];
  }

  // Constant tables, computed in double and rounded once to float32.
  const int ns = radar->n_samples, N = radar->fft_len, nb = d.info.n_bins;
  std::vector<float> win(ns);
  double wsum = 0.0;
  for (int t = 0; t < ns; ++t) {
    const double w = radar->range_window == 1 ? 0.5 - 0.5 * cos(2.0 * sar::kPi * t / (ns - 1)) : 1.0;
    win[t] = (float)w;
    wsum += w;
  }
  p->rc_scale = (float)(2.0 / wsum);  // one-sided spectrum of a real signal (A7)
  std::vector<float2> tw(std::max(1, N / 2));
  for (int q = 0; q < N / 2; ++q) {
    const double a = -2.0 * sar::kPi * (double)q / (double)N;
    tw[q] = make_float2((float)cos(a), (float)sin(a));
  }
  std::vector<float2> ramp(nb);
  const double tc = 0.5 * (ns - 1);
  for (int i = 0; i < nb; ++i) {
    const double k = (double)(d.info.k_lo + i);
    // exp(+j 2 pi k t_c / N); reduce k * t_c mod N exactly before scaling
    const double ph = fmod(k * tc, (double)N) / (double)N;
    ramp[i] = make_float2((float)cos(2.0 * sar::kPi * ph), (float)sin(2.0 * sar::kPi * ph));
  }
  // carrier phase of every crop bin's lower edge + half a bin: exp(j 2 pi beta (k + 1/2)),
  // beta = c2 / a1 cycles per bin (the BP kernel's phase folding, bp_kernel.cu); entry i
  // is crop bin i - 1 (from k = -1 up to n_bins - 1)
  std::vector<float2> bph(nb + 1);
  const double beta = d.info.c2_cycles_per_m / d.info.a1_bins_per_m;
  for (int i = 0; i <= nb; ++i) {
    double cyc = beta * ((double)(d.info.k_lo + i - 1) + 0.5);
    cyc -= floor(cyc);
    bph[i] = make_float2((float)cos(2.0 * sar::kPi * cyc), (float)sin(2.0 * sar::kPi * cyc));
  }
  // register-path range compression (rc_kernel.cu): per sub-transform b < N/L the window
  // times the pre-twiddle exp(-j 2 pi b t / N), and the Stockham stage twiddles W_64^(k r)
  // (k, r < 8) then W_L^(k r) (k < 64, r < R2 = L/64)
  const int rcL = sar::rc_path(ns, N, false);
  std::vector<float2> coef, stw;
  if (rcL) {
    const int zp = N / rcL, r2 = rcL / 64;
    coef.resize((size_t)zp * ns);
    for (int b = 0; b < zp; ++b)
      for (int t = 0; t < ns; ++t) {
        const double a = -2.0 * sar::kPi * (double)(((long long)b * t) % N) / (double)N;
        const double w = radar->range_window == 1 ? 0.5 - 0.5 * cos(2.0 * sar::kPi * t / (ns - 1)) : 1.0;
        coef[(size_t)b * ns + t] = make_float2((float)(w * cos(a)), (float)(w * sin(a)));
      }
    stw.resize(64 + 64 * r2);
    for (int k = 0; k < 8; ++k)
      for (int r = 0; r < 8; ++r) {
        const double a = -2.0 * sar::kPi * (double)(k * r) / 64.0;
        stw[k * 8 + r] = make_float2((float)cos(a), (float)sin(a));
      }
    for (int k = 0; k < 64; ++k)
      for (int r = 0; r < r2; ++r) {
        const double a = -2.0 * sar::kPi * (double)(k * r) / (double)rcL;
        stw[64 + k * r2 + r] = make_float2((float)cos(a), (float)sin(a));
      }
    if ((st = dev_alloc(&p->d_rc_coef, coef.size())) != SAR_OK || (st = dev_alloc(&p->d_rc_stw, stw.size())) != SAR_OK ||
        (e = cudaMemcpy(p->d_rc_coef, coef.data(), coef.size() * sizeof(float2), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(p->d_rc_stw, stw.data(), stw.size() * sizeof(float2), cudaMemcpyHostToDevice)) != cudaSuccess) {
      free_plan(p);
      return st != SAR_OK ? st : cuda_fail(e, "cudaMemcpy (range-compression tables)");
    }
  }
  if ((st = dev_alloc(&p->d_window, ns)) != SAR_OK || (st = dev_alloc(&p->d_twiddle, tw.size())) != SAR_OK ||
      (st = dev_alloc(&p->d_ramp, ramp.size())) != SAR_OK || (st = dev_alloc(&p->d_binphase, bph.size())) != SAR_OK) {
    free_plan(p);
    return st;
  }
  if ((e = cudaMemcpy(p->d_window, win.data(), ns * sizeof(float), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(p->d_twiddle, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(p->d_ramp, ramp.data(), ramp.size() * sizeof(float2), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(p->d_binphase, bph.data(), bph.size() * sizeof(float2), cudaMemcpyHostToDevice)) != cudaSuccess) {
    free_plan(p);
    return cuda_fail(e, "cudaMemcpy (plan tables)");
  }
  *out = p;
  return SAR_OK;
}

sar_status_t sar_plan_info(sar_plan_t plan, sar_plan_info_t* info) {
  if (!plan || !info) return fail(SAR_ERR_INVALID_ARGUMENT, "null argument");
  *info = plan->info;
  return SAR_OK;
}

sar_status_t sar_plan_crop(sar_plan_t plan, int32_t* k_lo, int32_t* n_bins) {
  if (!plan || !k_lo || !n_bins) return fail(SAR_ERR_INVALID_ARGUMENT, "null argument");
  *k_lo = plan->info.k_lo;
  *n_bins = plan->info.n_bins;
  return SAR_OK;
}

int64_t sar_plan_launch_count(sar_plan_t plan) { return plan ? plan->launches.load() : -1; }

sar_status_t sar_range_compress(sar_plan_t plan, const float* raw, const float* w_sar,
                                int32_t chirp0, int32_t nchirp, sar_complex64_t* profiles,
                                sar_stream_t stream) {
  if (!plan) return fail(SAR_ERR_INVALID_ARGUMENT, "plan is null");
  const sar_radar_params_t& r = plan->radar;
  if (chirp0 < 0 || nchirp < 0 || (int64_t)chirp0 + nchirp > r.n_chirps)
    return fail(SAR_ERR_INVALID_ARGUMENT, "chirp shard out of range");
  if (nchirp == 0) return SAR_OK;
  if (!raw || !profiles) return fail(SAR_ERR_INVALID_ARGUMENT, "raw and profiles must be non-null");
  DeviceGuard guard(plan->device);
  sar::RcArgs a;
  a.raw = raw;
  a.wsar = w_sar;
  a.window = plan->d_window;
  a.twiddle = plan->d_twiddle;
  a.coef = plan->d_rc_coef;
  a.stw = plan->d_rc_stw;
  a.ramp = plan->d_ramp;
  a.prof = reinterpret_cast<float2*>(profiles);
  a.row0 = chirp0 * r.n_rx;
  a.nrows = nchirp * r.n_rx;
  a.n_rx = r.n_rx;
  a.ns = r.n_samples;
  a.nfft = r.fft_len;
  a.log2n = 0;
  while ((1 << a.log2n) < r.fft_len) ++a.log2n;
  a.k_lo = plan->info.k_lo;
  a.n_bins = plan->info.n_bins;
  a.scale = plan->rc_scale;
  cudaError_t e = sar::launch_rc(a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "range compression launch");
  plan->launches.fetch_add(1);
  return SAR_OK;
}

namespace {
// A contiguous run of absolute tiles launched on one kernel family (near: the kernel with the
// per-tile near-field branch).
struct TileRun {
  int tile0, ntile;
  bool near;
};

// Would the BP kernel's per-tile near-field test (bp_kernel.cuh: anchor within 3 rho_T of the
// antenna box) take the SAFE form for tile (tx, ty)?  Same fp64 formulas, with a 0.1 % margin so
// that a tile the kernel would call near is never sent to the fast kernel.
bool tile_is_near(const sar_plan_t plan, int tx, int ty) {
  const int TX = plan->info.tile_x, TY = plan->info.tile_y;
  double pt[3], rho_t = plan->tile_rho;
  if (plan->polar) {
    const sar_polar_grid_t& pg = plan->pgrid;
    const double th = pg.th0 + (tx * TX + 0.5 * (TX - 1)) * pg.dth;
    const double rc = pg.r0 + (ty * TY + 0.5 * (TY - 1)) * pg.dr;
    pt[0] = pg.xc + rc * sin(th);
    pt[1] = pg.yc + rc * cos(th);
    pt[2] = pg.zc;
    const double ht = 0.5 * (TX - 1) * pg.dth, hr = 0.5 * (TY - 1) * pg.dr;
    rho_t = 0.0;
    for (int c = 0; c < 4; ++c) {
      const double rr = rc + ((c & 1) ? hr : -hr), dt = (c & 2) ? ht : -ht;
      rho_t = std::max(rho_t, sqrt(rr * rr + rc * rc - 2.0 * rr * rc * cos(dt)));
    }
  } else {
    const sar_grid_t& g = plan->grid;
    pt[0] = g.x0 + (tx * TX + 0.5 * (TX - 1)) * g.dx;
    pt[1] = g.y0 + (ty * TY + 0.5 * (TY - 1)) * g.dy;
    pt[2] = g.z0;
  }
  double d2 = 0.0;
  for (int k = 0; k < 3; ++k) {
    const double gap = std::max(0.0, std::max(plan->box.lo[k] - pt[k], pt[k] - plan->box.hi[k]));
    d2 += gap * gap;
  }
  const double near_r = (3.0 * rho_t * (1.0 + 1e-6) + 1e-3) * 1.001 + 1e-6;
  return d2 < near_r * near_r;
}

// Split [tile0, tile0 + ntile) into runs of near-field / far-field tiles (plans without
// near-field tiles: one far run).  Many short runs (an antenna box inside the grid) fall back
// to one run on the near-field kernel, which tests every tile itself.
std::vector<TileRun> tile_runs(const sar_plan_t plan, int tile0, int ntile, int tiles_x) {
  std::vector<TileRun> runs;
  if (!plan->near_field) {
    runs.push_back({tile0, ntile, false});
    return runs;
  }
  for (int t = tile0; t < tile0 + ntile; ++t) {
    const bool nr = tile_is_near(plan, t % tiles_x, t / tiles_x);
    if (!runs.empty() && runs.back().near == nr) ++runs.back().ntile;
    else runs.push_back({t, 1, nr});
  }
  if (runs.size() > 8) runs.assign(1, TileRun{tile0, ntile, true});
  return runs;
}

sar_status_t backproject_impl(sar_plan_t plan, const sar_complex64_t* profiles, const double* tx_pos,
                              const double* rx_pos, const float* doppler_bins, int32_t chirp0,
                              int32_t nchirp, int32_t row0, int32_t nrow, sar_complex64_t* image,
                              int32_t accumulate, sar_complex64_t* const* peers, int32_t n_peer,
                              int32_t multicast, sar_stream_t stream, int32_t tile0 = -1, int32_t ntile = 0) {
  // Row mode (tile0 < 0): rows [row0, row0 + nrow), the CTAs run every absolute grid tile those
  // rows touch.  Tile mode: the absolute tiles [tile0, tile0 + ntile); `image` is the full
  // [ny][nx] image and the call writes the pixels of those tiles only.
  if (!plan) return fail(SAR_ERR_INVALID_ARGUMENT, "plan is null");
  const sar_radar_params_t& r = plan->radar;
  const sar_grid_t& g = plan->grid;
  const int TXp = plan->info.tile_x, TYp = plan->info.tile_y;
  const int tiles_x = (g.nx + TXp - 1) / TXp, tiles_y = (g.ny + TYp - 1) / TYp;
  if (chirp0 < 0 || nchirp < 0 || (int64_t)chirp0 + nchirp > r.n_chirps)
    return fail(SAR_ERR_INVALID_ARGUMENT, "chirp shard out of range");
  if (tile0 >= 0) {
    if (ntile < 0 || (int64_t)tile0 + ntile > (int64_t)tiles_x * tiles_y)
      return fail(SAR_ERR_INVALID_ARGUMENT, "tile range out of range");
    if (ntile == 0) return SAR_OK;
    const int ty0 = tile0 / tiles_x, ty1 = (tile0 + ntile - 1) / tiles_x;
    row0 = ty0 * TYp;
    nrow = std::min(g.ny, (ty1 + 1) * TYp) - row0;
    if (image) image += (size_t)row0 * g.nx;
  } else {
    if (row0 < 0 || nrow < 0 || (int64_t)row0 + nrow > g.ny)
      return fail(SAR_ERR_INVALID_ARGUMENT, "row shard out of range");
    if (nrow > 0) {
      tile0 = (row0 / TYp) * tiles_x;
      ntile = ((row0 + nrow - 1) / TYp + 1) * tiles_x - tile0;
    }
  }
  if (accumulate != 0 && accumulate != 1) return fail(SAR_ERR_INVALID_ARGUMENT, "accumulate must be 0 or 1");
  if (!rx_pos && r.n_rx != 1)
    return fail(SAR_ERR_INVALID_ARGUMENT, "rx_pos may be NULL (monostatic) only when n_rx == 1");
  if (doppler_bins && !(r.doppler_max_bins > 0.0f))
    return fail(SAR_ERR_INVALID_ARGUMENT, "a Doppler array needs doppler_max_bins > 0 in the plan");
  if (nrow == 0 || (nchirp == 0 && accumulate)) return SAR_OK;
  if (!image || (nchirp > 0 && (!profiles || !tx_pos)))
    return fail(SAR_ERR_INVALID_ARGUMENT, "image, profiles and tx_pos must be non-null");
  DeviceGuard guard(plan->device);
  sar::BpArgs a;
  a.prof = reinterpret_cast<const float2*>(profiles);
  a.tx = tx_pos;
  a.rx = rx_pos;
  a.dop = doppler_bins;
  a.img = reinterpret_cast<float2*>(image);
  a.n_bins = plan->info.n_bins;
  a.n_rx = r.n_rx;
  a.chirp0 = chirp0;
  a.nchirp = nchirp;
  a.row0 = row0;
  a.nrow = nrow;
  a.nx = g.nx;
  a.tiles_x = tiles_x;   // (tile ranges per launch below)
  a.S = plan->bp_stages;
  a.ncw = plan->bp_ncw;
  a.pb = plan->bp_pb;
  a.accumulate = accumulate;
  a.W = plan->info.window_bins;
  {   // tuning / test switch, read per call: SAR_BP_DERIVE=0 keeps one rsqrt leg per chirp
    const char* e = getenv("SAR_BP_DERIVE");
    a.derive = e && e[0] == '0' ? 0 : 1;
  }
  a.dop_max = r.doppler_max_bins;
  a.CB = plan->info.chirps_per_stage;
  a.x0 = g.x0;
  a.y0 = g.y0;
  a.z0 = g.z0;
  a.dx = g.dx;
  a.dy = g.dy;
  a.polar = plan->polar ? 1 : 0;
  a.r0 = plan->pgrid.r0;
  a.dr = plan->pgrid.dr;
  a.th0 = plan->pgrid.th0;
  a.dth = plan->pgrid.dth;
  a.a1 = plan->info.a1_bins_per_m;
  a.c2 = plan->info.c2_cycles_per_m;
  a.k_lo = plan->info.k_lo;
  a.kap_half = plan->info.window_half_bins;
  for (int k = 0; k < 3; ++k) {
    a.box_lo[k] = plan->box.lo[k];
    a.box_hi[k] = plan->box.hi[k];
  }
  a.tile_rho = plan->tile_rho;
  const bool bistatic = rx_pos != nullptr;
  a.A1f = (float)(bistatic ? a.a1 : 2.0 * a.a1);
  a.binphase = plan->d_binphase;
  a.C3f = (float)(2.0 * sar::kPi * a.c2 / a.a1);
  a.n_peer = n_peer;
  a.multicast = multicast;
  a.split_query = nullptr;
  a.ksplit_out = nullptr;
  a.pairs = nullptr;
  a.pair_stride = a.pair_pad = 0;
  float4* pairs = nullptr;
  static const bool no_pairs = [] {   // test switch: the producer builds the windows itself
    const char* e = getenv("SAR_BP_NO_PAIRS");
    return e && e[0] == '1';
  }();
  // Pair rows cover the bins of this call's tiles only (a shard's own crop over the rows of
  // the tiles it runs, whole tiles included, same margins as the plan's)
  int kb0 = 0, kbn = plan->info.n_bins;
  const int trow0 = (tile0 / tiles_x) * TYp;
  const int trow1 = std::min(g.ny, ((tile0 + ntile - 1) / tiles_x + 1) * TYp);
  if (trow0 != 0 || trow1 != g.ny) {
    sar_grid_t sg = g;
    sar_polar_grid_t spg = plan->pgrid;
    if (plan->polar) {
      spg.r0 = plan->pgrid.r0 + trow0 * plan->pgrid.dr;
      spg.n_r = trow1 - trow0;
    } else {
      sg.y0 = g.y0 + trow0 * g.dy;
    }
    sg.ny = trow1 - trow0;
    double dmin, dmax;
    long lo, hi;
    if (crop_bins(&r, &sg, &plan->box, plan->polar ? &spg : nullptr, plan->info.a1_bins_per_m, &dmin, &dmax, &lo,
                  &hi) == SAR_OK) {
      const long b0 = std::max(0L, std::min(lo - plan->info.k_lo, (long)plan->info.n_bins));
      const long b1 = std::max(b0, std::min(hi - plan->info.k_lo + 1, (long)plan->info.n_bins));
      kb0 = (int)b0;
      kbn = (int)(b1 - b0);
    }
  }
  if (nchirp > 0 && !no_pairs) {
    // Pair-format rows of this call's chirps (pair_kernel, HBM-bound), in a stream-ordered
    // allocation from the plan's pool so that calls on different streams stay independent;
    // the BP producer then only issues one bulk copy per (tile, chirp, RX) window.
    const int pad = plan->info.window_bins + 2, stride = kbn + 2 * pad;
    const size_t rows = (size_t)nchirp * r.n_rx;
    cudaError_t pe = cudaMallocFromPoolAsync((void**)&pairs, rows * stride * sizeof(float4), plan->pool,
                                             (cudaStream_t)stream);
    if (pe != cudaSuccess) {   // no room for the rows: the producer builds the windows itself
      cudaGetLastError();
      pairs = nullptr;
    }
  }
  if (pairs) {
    const int pad = plan->info.window_bins + 2, stride = kbn + 2 * pad;
    const size_t rows = (size_t)nchirp * r.n_rx;
    sar::PairArgs pa;
    pa.prof = a.prof + (size_t)chirp0 * r.n_rx * plan->info.n_bins;
    pa.binphase = plan->d_binphase;
    pa.out = pairs;
    pa.row0 = 0;
    pa.rows = (int)rows;
    pa.n_bins = plan->info.n_bins;
    pa.stride = stride;
    pa.pad = pad;
    pa.k0 = kb0;
    cudaError_t pe = sar::launch_pairs(pa, (cudaStream_t)stream);
    if (pe != cudaSuccess) {
      cudaFreeAsync(pairs, (cudaStream_t)stream);
      return cuda_fail(pe, "pair-format launch");
    }
    a.pairs = pairs - (size_t)chirp0 * r.n_rx * stride;   // indexed by absolute (chirp, RX) row
    a.pair_stride = stride;
    a.pair_pad = pad - kb0;
  }
  for (int d = 0; d < 8; ++d) a.peer[d] = d < n_peer ? reinterpret_cast<float2*>(peers[d]) : nullptr;
  static const bool scatter_nosplit = [] {   // tuning switch: scatters always unsplit
    const char* e = getenv("SAR_BP_SCATTER_NOSPLIT");
    return e && e[0] == '1';
  }();
  // One launch per run of tiles: a plan with near-field tiles runs them (and only them) on the
  // kernel with the per-tile SAFE branch; every other tile runs on the fast kernel (C0: near-field
  // rows 18.3 -> 13.0 ms in round 1 by the per-tile branch; separate launches 10.48 -> 9.95 ms).
  std::vector<TileRun> runs = tile_runs(plan, tile0, ntile, tiles_x);
  cudaError_t e = cudaSuccess;
  int64_t launched = pairs ? 1 : 0;
  // (the runs share the caller's stream: a side stream for the near-field runs measured no faster
  //  on C0 with the L2 flushed between steps, and its step time varied by +-3 %)
  for (const TileRun& run : runs) {
    void* const rstream = stream;
    sar::BpArgs b = a;
    b.ty0 = run.tile0 / tiles_x;   // the launch covers whole tile rows; [tile_lo, tile_hi) compute
    b.tile_lo = run.tile0 - b.ty0 * tiles_x;
    b.tile_hi = b.tile_lo + run.ntile;
    b.ntile = ((run.tile0 + run.ntile - 1) / tiles_x + 1) * tiles_x - b.ty0 * tiles_x;
    b.ws = nullptr;
    b.ws_plane = 0;
    b.ws_planes = 0;
    b.tile_count = nullptr;
    // rows of this run inside the call's image rows (the chunk planes cover only those)
    const int rr0 = std::max(0, b.ty0 * TYp - row0);
    const int rr1 = std::min(nrow, (b.ty0 + b.ntile / tiles_x) * TYp - row0);
    float2* ws_buf = nullptr;
    if (nchirp > 0 && !(n_peer > 0 && scatter_nosplit)) {
      // a launch that would run chirp-split: one workspace plane per chunk (+ per-tile counters
      // for a scatter, whose last chunk per tile publishes it) from the plan's pool; without
      // them it runs unsplit
      int k = 1;
      sar::BpArgs q = b;   // the launcher's split of this launch (its scatter policy included)
      q.split_query = &k;
      if (sar::launch_bp(q, bistatic, doppler_bins != nullptr, run.near, (cudaStream_t)rstream) == cudaSuccess &&
          k > 1) {
        b.ws_plane = (long)(rr1 - rr0) * g.nx;
        const int planes = n_peer > 0 ? k : k - 1;   // a plain launch keeps chunk 0 in the image
        if (cudaMallocFromPoolAsync((void**)&ws_buf, (size_t)planes * b.ws_plane * sizeof(float2), plan->pool,
                                    (cudaStream_t)rstream) != cudaSuccess ||
            (n_peer > 0 && cudaMallocFromPoolAsync((void**)&b.tile_count, (size_t)b.ntile * sizeof(int), plan->pool,
                                                   (cudaStream_t)rstream) != cudaSuccess)) {
          cudaGetLastError();
          if (ws_buf) cudaFreeAsync(ws_buf, (cudaStream_t)rstream);
          ws_buf = nullptr;
          b.tile_count = nullptr;
        } else {
          // planes indexed by the image row (kernel and split sum): offset to the run's rows
          b.ws = ws_buf - (ptrdiff_t)rr0 * g.nx;
          b.ws_planes = planes;
        }
      }
    }
    int ksplit = 1;
    b.ksplit_out = &ksplit;
    e = sar::launch_bp(b, bistatic, doppler_bins != nullptr, run.near, (cudaStream_t)rstream);
    if (e == cudaSuccess) ++launched;
    if (e == cudaSuccess && ksplit > 1 && n_peer == 0) {
      // the chunk planes in chunk order into the image (deterministic)
      sar::SplitSumArgs sa;
      sa.img = b.img;
      sa.ws = b.ws;
      sa.plane = b.ws_plane;
      sa.planes = ksplit - 1;
      sa.tile0 = run.tile0;
      sa.ntile = run.ntile;
      sa.tiles_x = tiles_x;
      sa.tile_y = TYp;
      sa.row0 = row0;
      sa.nrow = nrow;
      sa.nx = g.nx;
      e = sar::launch_split_sum(sa, (cudaStream_t)rstream);
      if (e == cudaSuccess) ++launched;
    }
    if (ws_buf) cudaFreeAsync(ws_buf, (cudaStream_t)rstream);
    if (b.tile_count) cudaFreeAsync(b.tile_count, (cudaStream_t)rstream);
    if (e != cudaSuccess) break;
  }
  if (pairs) cudaFreeAsync(pairs, (cudaStream_t)stream);
  plan->launches.fetch_add(launched);
  if (e != cudaSuccess) return cuda_fail(e, "back-projection launch");
  return SAR_OK;
}
}  // namespace

sar_status_t sar_backproject(sar_plan_t plan, const sar_complex64_t* profiles,
                             const double* tx_pos, const double* rx_pos,
                             const float* doppler_bins, int32_t chirp0, int32_t nchirp,
                             int32_t row0, int32_t nrow, sar_complex64_t* image,
                             int32_t accumulate, sar_stream_t stream) {
  return backproject_impl(plan, profiles, tx_pos, rx_pos, doppler_bins, chirp0, nchirp, row0, nrow, image,
                          accumulate, nullptr, 0, 0, stream);
}

sar_status_t sar_backproject_scatter(sar_plan_t plan, const sar_complex64_t* profiles,
                                     const double* tx_pos, const double* rx_pos,
                                     const float* doppler_bins, int32_t chirp0, int32_t nchirp,
                                     int32_t row0, int32_t nrow, sar_complex64_t* const* images,
                                     int32_t n_images, int32_t flags, sar_stream_t stream) {
  if (!images || n_images < 1 || n_images > 8)
    return fail(SAR_ERR_INVALID_ARGUMENT, "images must hold 1..8 device pointers");
  if (flags & ~(SAR_SCATTER_MULTICAST | SAR_SCATTER_ADD)) return fail(SAR_ERR_INVALID_ARGUMENT, "unknown flags");
  const int multicast = (flags & SAR_SCATTER_MULTICAST) ? 1 : 0, add = (flags & SAR_SCATTER_ADD) ? 1 : 0;
  if (multicast && n_images != 1)
    return fail(SAR_ERR_INVALID_ARGUMENT, "a multicast store takes exactly one (multicast) address");
  for (int d = 0; d < n_images; ++d)
    if (!images[d]) return fail(SAR_ERR_INVALID_ARGUMENT, "null image pointer");
  if (add && nchirp == 0) return SAR_OK;
  return backproject_impl(plan, profiles, tx_pos, rx_pos, doppler_bins, chirp0, nchirp, row0, nrow, images[0],
                          add, images, n_images, multicast, stream);
}

sar_status_t sar_backproject_tiles(sar_plan_t plan, const sar_complex64_t* profiles, const double* tx_pos,
                                   const double* rx_pos, const float* doppler_bins, int32_t chirp0,
                                   int32_t nchirp, int32_t tile0, int32_t ntile, sar_complex64_t* image,
                                   int32_t accumulate, sar_stream_t stream) {
  if (tile0 < 0) return fail(SAR_ERR_INVALID_ARGUMENT, "tile0 must be >= 0");
  return backproject_impl(plan, profiles, tx_pos, rx_pos, doppler_bins, chirp0, nchirp, 0, 0, image, accumulate,
                          nullptr, 0, 0, stream, tile0, ntile);
}

sar_status_t sar_backproject_scatter_tiles(sar_plan_t plan, const sar_complex64_t* profiles,
                                           const double* tx_pos, const double* rx_pos,
                                           const float* doppler_bins, int32_t chirp0, int32_t nchirp,
                                           int32_t tile0, int32_t ntile, sar_complex64_t* const* images,
                                           int32_t n_images, int32_t flags, sar_stream_t stream) {
  if (tile0 < 0) return fail(SAR_ERR_INVALID_ARGUMENT, "tile0 must be >= 0");
  if (!images || n_images < 1 || n_images > 8)
    return fail(SAR_ERR_INVALID_ARGUMENT, "images must hold 1..8 device pointers");
  if (flags & ~(SAR_SCATTER_MULTICAST | SAR_SCATTER_ADD | SAR_SCATTER_PUBLISH))
    return fail(SAR_ERR_INVALID_ARGUMENT, "unknown flags");
  if (flags & SAR_SCATTER_PUBLISH) {
    if (flags & (SAR_SCATTER_MULTICAST | SAR_SCATTER_ADD))
      return fail(SAR_ERR_INVALID_ARGUMENT, "SAR_SCATTER_PUBLISH stores only, to P2P images");
    for (int d = 0; d < n_images; ++d)
      if (!images[d]) return fail(SAR_ERR_INVALID_ARGUMENT, "null image pointer");
    // the tiles into the caller's own image, then one copy of them to every other image
    sar_status_t st = backproject_impl(plan, profiles, tx_pos, rx_pos, doppler_bins, chirp0, nchirp, 0, 0, images[0],
                                       0, nullptr, 0, 0, stream, tile0, ntile);
    if (st != SAR_OK || ntile == 0 || n_images == 1) return st;
    DeviceGuard guard(plan->device);
    const sar_grid_t& g = plan->grid;
    sar::PublishArgs pa;
    pa.src = reinterpret_cast<const float2*>(images[0]);
    for (int d = 0; d < 8; ++d) pa.dst[d] = d + 1 < n_images ? reinterpret_cast<float2*>(images[d + 1]) : nullptr;
    pa.n_dst = n_images - 1;
    pa.tile0 = tile0;
    pa.ntile = ntile;
    pa.tiles_x = (g.nx + plan->info.tile_x - 1) / plan->info.tile_x;
    pa.tile_y = plan->info.tile_y;
    pa.nx = g.nx;
    pa.ny = g.ny;
    cudaError_t e = sar::launch_publish(pa, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "publish launch");
    plan->launches.fetch_add(1);
    return SAR_OK;
  }
  const int multicast = (flags & SAR_SCATTER_MULTICAST) ? 1 : 0, add = (flags & SAR_SCATTER_ADD) ? 1 : 0;
  if (multicast && n_images != 1)
    return fail(SAR_ERR_INVALID_ARGUMENT, "a multicast store takes exactly one (multicast) address");
  for (int d = 0; d < n_images; ++d)
    if (!images[d]) return fail(SAR_ERR_INVALID_ARGUMENT, "null image pointer");
  if (add && nchirp == 0) return SAR_OK;
  return backproject_impl(plan, profiles, tx_pos, rx_pos, doppler_bins, chirp0, nchirp, 0, 0, images[0], add,
                          images, n_images, multicast, stream, tile0, ntile);
}

sar_status_t sar_plan_tiles(sar_plan_t plan, int32_t* tiles_x, int32_t* tiles_y) {
  if (!plan || !tiles_x || !tiles_y) return fail(SAR_ERR_INVALID_ARGUMENT, "null argument");
  *tiles_x = (plan->grid.nx + plan->info.tile_x - 1) / plan->info.tile_x;
  *tiles_y = (plan->grid.ny + plan->info.tile_y - 1) / plan->info.tile_y;
  return SAR_OK;
}

#ifndef SAR_FORM_BANDS
// sar_form_image: bands of the readback pipeline (0: the BP epilogue stores into the host image).
// Measured (tools/gpu_r4t.sh) e2e with 0 / 2 / 4 / 8 bands: C3 51.55 / 51.24 / 51.04 / 51.41 ms; C4
// 891.7 (0) / 882.4 (4) ms: the epilogue's host stores kept the launch unsplit (no L2 window for
// scatters), the bands run the plain kernels
#define SAR_FORM_BANDS 4
#endif
constexpr int kFormBands = SAR_FORM_BANDS;

sar_status_t sar_form_image(sar_plan_t plan, const float* raw_host, const float* w_sar_host,
                            const double* tx_host, const double* rx_host,
                            const float* doppler_host, int32_t row0, int32_t nrow,
                            sar_complex64_t* image_host, sar_stream_t stream) {
  if (!plan) return fail(SAR_ERR_INVALID_ARGUMENT, "plan is null");
  const sar_radar_params_t& r = plan->radar;
  const sar_grid_t& g = plan->grid;
  if (row0 < 0 || nrow < 0 || (int64_t)row0 + nrow > g.ny)
    return fail(SAR_ERR_INVALID_ARGUMENT, "row shard out of range");
  if (!raw_host || !tx_host || !image_host)
    return fail(SAR_ERR_INVALID_ARGUMENT, "raw_host, tx_host and image_host must be non-null");
  if (!rx_host && r.n_rx != 1)
    return fail(SAR_ERR_INVALID_ARGUMENT, "rx_host may be NULL only when n_rx == 1");
  // Coverage check of the declared antenna box (the crop relies on it).
  const double tol = 1e-9;
  auto inside = [&](const double* q) {
    for (int k = 0; k < 3; ++k)
      if (!(q[k] >= plan->box.lo[k] - tol && q[k] <= plan->box.hi[k] + tol)) return false;
    return true;
  };
  for (int m = 0; m < r.n_chirps; ++m) {
    if (!inside(tx_host + 3 * (size_t)m))
      return fail(SAR_ERR_OUT_OF_COVERAGE, "a TX position lies outside the declared antenna box");
    if (rx_host)
      for (int n = 0; n < r.n_rx; ++n)
        if (!inside(rx_host + 3 * ((size_t)m * r.n_rx + n)))
          return fail(SAR_ERR_OUT_OF_COVERAGE, "an RX position lies outside the declared antenna box");
  }
  DeviceGuard guard(plan->device);
  const size_t M = r.n_chirps, R = r.n_rx, NS = r.n_samples, NB = plan->info.n_bins;
  const size_t npix = (size_t)g.nx * g.ny;
  sar_status_t st;
  std::lock_guard<std::mutex> ws_lock(plan->ws_mutex);
  if (!plan->w_img) {   // w_img is allocated last: non-null means the whole workspace exists
    if ((st = dev_alloc(&plan->w_raw, M * R * NS)) != SAR_OK || (st = dev_alloc(&plan->w_wsar, M)) != SAR_OK ||
        (st = dev_alloc(&plan->w_tx, M * 3)) != SAR_OK || (st = dev_alloc(&plan->w_rx, M * R * 3)) != SAR_OK ||
        (st = dev_alloc(&plan->w_dop, npix)) != SAR_OK || (st = dev_alloc(&plan->w_prof, M * R * NB)) != SAR_OK ||
        (st = dev_alloc(&plan->w_img, npix)) != SAR_OK) {
      cudaFree(plan->w_raw); cudaFree(plan->w_wsar); cudaFree(plan->w_tx); cudaFree(plan->w_rx);
      cudaFree(plan->w_dop); cudaFree(plan->w_prof);
      plan->w_raw = nullptr; plan->w_wsar = nullptr; plan->w_tx = nullptr; plan->w_rx = nullptr;
      plan->w_dop = nullptr; plan->w_prof = nullptr; plan->w_img = nullptr;
      return st;
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  // Raw samples are read exactly once, by the range compression: from a pinned (device-mapped)
  // host buffer the kernel reads them over the host link directly (no staging copy); poses,
  // re-read by every BP tile, are copied.
  void* raw_mapped = nullptr;
  const bool raw_direct = cudaHostGetDevicePointer(&raw_mapped, const_cast<float*>(raw_host), 0) == cudaSuccess &&
                          raw_mapped;
  if (!raw_direct) cudaGetLastError();
  if ((!raw_direct &&
       (e = cudaMemcpyAsync(plan->w_raw, raw_host, M * R * NS * sizeof(float), cudaMemcpyHostToDevice, s)) != cudaSuccess) ||
      (e = cudaMemcpyAsync(plan->w_tx, tx_host, M * 3 * sizeof(double), cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync H2D");
  if (w_sar_host && (e = cudaMemcpyAsync(plan->w_wsar, w_sar_host, M * sizeof(float), cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync H2D");
  if (rx_host && (e = cudaMemcpyAsync(plan->w_rx, rx_host, M * R * 3 * sizeof(double), cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync H2D");
  if (doppler_host && (e = cudaMemcpyAsync(plan->w_dop, doppler_host, npix * sizeof(float), cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync H2D");
  st = sar_range_compress(plan, raw_direct ? static_cast<const float*>(raw_mapped) : plan->w_raw,
                          w_sar_host ? plan->w_wsar : nullptr, 0, r.n_chirps,
                          reinterpret_cast<sar_complex64_t*>(plan->w_prof), stream);
  if (st != SAR_OK) return st;
  // Image readback fused into the BP epilogue: when the host image is pinned (device-mapped
  // under UVA) every finished tile is stored straight into host memory while the other tiles
  // compute (under a chirp split by the last chunk of
  // each tile from an accumulation image);
  // else one device->host copy after the kernel.
  void* mapped = nullptr;
  const bool direct = nrow > 0 && cudaHostGetDevicePointer(&mapped, image_host, 0) == cudaSuccess && mapped;
  if (!direct) cudaGetLastError();   // clear the error of a pageable buffer
  static const int bands_env = [] {   // SAR_FORM_BANDS=n: banded readback pipeline (0: epilogue stores)
    const char* v = getenv("SAR_FORM_BANDS");
    return v && *v ? atoi(v) : kFormBands;
  }();
  const int TYp = plan->info.tile_y;
  const int trow0 = row0 / TYp, trow1 = (row0 + nrow + TYp - 1) / TYp;
  // bands only where each still fills the GPU twice over (~3 resident CTAs per SM): small grids
  // lose more to per-band tails than the overlap saves (C0 / C6, 1444 tiles: e2e +1.4 % / +5 %)
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, plan->device);
  const int64_t call_tiles = (int64_t)(trow1 - trow0) * ((g.nx + plan->info.tile_x - 1) / plan->info.tile_x);
  const int nbands = (int)std::min<int64_t>(std::min(std::min(bands_env, 8), trow1 - trow0),
                                            call_tiles / (2 * 3 * (int64_t)sms));
  if (direct && nbands >= 2) {
    // Readback pipelined with the compute: the call's rows run as bands of whole tile rows; each
    // band's BP writes the plan's device image (plain kernels, L2-bounded chirp split), then the
    // band is copied to the pinned host image on the plan's copy stream while the next band
    // computes; `stream` waits for the last copy.
    if (!plan->w_copy) {
      if ((e = cudaStreamCreateWithFlags(&plan->w_copy, cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_fail(e, "copy stream");
      for (cudaEvent_t& ev : plan->w_ev)
        if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e, "event");
    }
    for (int bnd = 0; bnd < nbands; ++bnd) {
      const int tb0 = trow0 + (int)((int64_t)(trow1 - trow0) * bnd / nbands);
      const int tb1 = trow0 + (int)((int64_t)(trow1 - trow0) * (bnd + 1) / nbands);
      const int rb0 = std::max(row0, tb0 * TYp), rb1 = std::min(row0 + nrow, tb1 * TYp);
      if (rb1 <= rb0) continue;
      st = sar_backproject(plan, reinterpret_cast<sar_complex64_t*>(plan->w_prof), plan->w_tx,
                           rx_host ? plan->w_rx : nullptr, doppler_host ? plan->w_dop : nullptr, 0, r.n_chirps,
                           rb0, rb1 - rb0, reinterpret_cast<sar_complex64_t*>(plan->w_img) + (size_t)(rb0 - row0) * g.nx,
                           0, stream);
      if (st != SAR_OK) return st;
      if ((e = cudaEventRecord(plan->w_ev[bnd], s)) != cudaSuccess ||
          (e = cudaStreamWaitEvent(plan->w_copy, plan->w_ev[bnd], 0)) != cudaSuccess ||
          (e = cudaMemcpyAsync(image_host + (size_t)(rb0 - row0) * g.nx, plan->w_img + (size_t)(rb0 - row0) * g.nx,
                               (size_t)(rb1 - rb0) * g.nx * sizeof(float2), cudaMemcpyDeviceToHost, plan->w_copy)) !=
              cudaSuccess)
        return cuda_fail(e, "band readback");
    }
    if ((e = cudaEventRecord(plan->w_ev[8], plan->w_copy)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(s, plan->w_ev[8], 0)) != cudaSuccess)
      return cuda_fail(e, "readback join");
    return SAR_OK;
  }
  if (direct) {
    sar_complex64_t* base = reinterpret_cast<sar_complex64_t*>(mapped) - (ptrdiff_t)row0 * g.nx;
    return backproject_impl(plan, reinterpret_cast<sar_complex64_t*>(plan->w_prof), plan->w_tx,
                            rx_host ? plan->w_rx : nullptr, doppler_host ? plan->w_dop : nullptr, 0, r.n_chirps,
                            row0, nrow, base, 0, &base, 1, 0, stream);
  }
  st = sar_backproject(plan, reinterpret_cast<sar_complex64_t*>(plan->w_prof), plan->w_tx,
                       rx_host ? plan->w_rx : nullptr, doppler_host ? plan->w_dop : nullptr, 0,
                       r.n_chirps, row0, nrow, reinterpret_cast<sar_complex64_t*>(plan->w_img), 0, stream);
  if (st != SAR_OK) return st;
  if (nrow > 0 &&
      (e = cudaMemcpyAsync(image_host, plan->w_img, (size_t)nrow * g.nx * sizeof(float2), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync D2H");
  return SAR_OK;
}

sar_status_t sar_doppler_table(const sar_radar_params_t* radar, const sar_grid_t* grid,
                               const double q_ref[3], const double v_avg[3], float* doppler_bins,
                               sar_stream_t stream) {
  if (!radar || !grid || !q_ref || !v_avg || !doppler_bins)
    return fail(SAR_ERR_INVALID_ARGUMENT, "null argument");
  if (!finite_pos(radar->f0_hz) || !finite_pos(radar->sample_rate_hz) || radar->fft_len < 1)
    return fail(SAR_ERR_INVALID_ARGUMENT, "f0_hz, sample_rate_hz and fft_len must be positive");
  if (!finite_pos(grid->dx) || !finite_pos(grid->dy) || grid->nx < 1 || grid->ny < 1)
    return fail(SAR_ERR_INVALID_ARGUMENT, "grid needs dx, dy > 0 and nx, ny >= 1");
  for (int k = 0; k < 3; ++k)
    if (!isfinite(q_ref[k]) || !isfinite(v_avg[k])) return fail(SAR_ERR_INVALID_ARGUMENT, "non-finite q_ref/v_avg");
  sar::DopArgs a{};
  a.out = doppler_bins;
  a.x0 = grid->x0;
  a.y0 = grid->y0;
  a.z0 = grid->z0;
  a.dx = grid->dx;
  a.dy = grid->dy;
  a.nx = grid->nx;
  a.ny = grid->ny;
  for (int k = 0; k < 3; ++k) {
    a.q[k] = q_ref[k];
    a.v[k] = v_avg[k];
  }
  a.legs = 2.0;
  a.bins_per_mps = radar->f0_hz / sar::kLightSpeed / (radar->sample_rate_hz / radar->fft_len);
  cudaError_t e = sar::launch_doppler(a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "doppler table launch");
  return SAR_OK;
}

sar_status_t sar_doppler_table_polar(const sar_radar_params_t* radar, const sar_polar_grid_t* grid,
                                     const double q_ref[3], const double v_avg[3], float* doppler_bins,
                                     sar_stream_t stream) {
  if (!radar || !grid || !q_ref || !v_avg || !doppler_bins)
    return fail(SAR_ERR_INVALID_ARGUMENT, "null argument");
  if (!finite_pos(radar->f0_hz) || !finite_pos(radar->sample_rate_hz) || radar->fft_len < 1)
    return fail(SAR_ERR_INVALID_ARGUMENT, "f0_hz, sample_rate_hz and fft_len must be positive");
  double lo[3], hi[3];
  sar_grid_t stand_in;
  sar_status_t st = polar_box(grid, lo, hi, &stand_in);
  if (st != SAR_OK) return st;
  for (int k = 0; k < 3; ++k)
    if (!isfinite(q_ref[k]) || !isfinite(v_avg[k])) return fail(SAR_ERR_INVALID_ARGUMENT, "non-finite q_ref/v_avg");
  sar::DopArgs a{};
  a.out = doppler_bins;
  a.x0 = grid->xc;
  a.y0 = grid->yc;
  a.z0 = grid->zc;
  a.nx = grid->n_th;
  a.ny = grid->n_r;
  a.polar = 1;
  a.r0 = grid->r0;
  a.dr = grid->dr;
  a.th0 = grid->th0;
  a.dth = grid->dth;
  for (int k = 0; k < 3; ++k) {
    a.q[k] = q_ref[k];
    a.v[k] = v_avg[k];
  }
  a.legs = 2.0;
  a.bins_per_mps = radar->f0_hz / sar::kLightSpeed / (radar->sample_rate_hz / radar->fft_len);
  cudaError_t e = sar::launch_doppler(a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "doppler table launch");
  return SAR_OK;
}

sar_status_t sar_polar_to_cartesian(const sar_polar_grid_t* polar, const sar_complex64_t* polar_image,
                                    const sar_grid_t* cart, sar_complex64_t* out, sar_stream_t stream) {
  if (!polar || !polar_image || !cart || !out) return fail(SAR_ERR_INVALID_ARGUMENT, "null argument");
  double lo[3], hi[3];
  sar_grid_t stand_in;
  sar_status_t st = polar_box(polar, lo, hi, &stand_in);
  if (st != SAR_OK) return st;
  if (!finite_pos(cart->dx) || !finite_pos(cart->dy) || cart->nx < 1 || cart->ny < 1)
    return fail(SAR_ERR_INVALID_ARGUMENT, "Cartesian grid needs dx, dy > 0 and nx, ny >= 1");
  sar::ResampleArgs a;
  a.in = reinterpret_cast<const float2*>(polar_image);
  a.out = reinterpret_cast<float2*>(out);
  a.xc = polar->xc;
  a.yc = polar->yc;
  a.r0 = polar->r0;
  a.dr = polar->dr;
  a.th0 = polar->th0;
  a.dth = polar->dth;
  a.n_th = polar->n_th;
  a.n_r = polar->n_r;
  a.x0 = cart->x0;
  a.y0 = cart->y0;
  a.dx = cart->dx;
  a.dy = cart->dy;
  a.nx = cart->nx;
  a.ny = cart->ny;
  cudaError_t e = sar::launch_resample(a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "polar-to-Cartesian launch");
  return SAR_OK;
}

sar_status_t sar_image_sum(sar_complex64_t* out, const sar_complex64_t* partials, int32_t n_partials,
                           int64_t stride, int64_t n_elems, sar_stream_t stream) {
  if (!out || !partials) return fail(SAR_ERR_INVALID_ARGUMENT, "null argument");
  if (n_partials < 1 || n_elems < 0 || stride < n_elems)
    return fail(SAR_ERR_INVALID_ARGUMENT, "need n_partials >= 1 and stride >= n_elems >= 0");
  if (n_elems == 0) return SAR_OK;
  cudaError_t e = sar::launch_sum(reinterpret_cast<float2*>(out), reinterpret_cast<const float2*>(partials),
                                  n_partials, (long)stride, (long)n_elems, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "image sum launch");
  return SAR_OK;
}

sar_status_t sar_destroy(sar_plan_t plan) {
  if (!plan) return fail(SAR_ERR_INVALID_ARGUMENT, "plan is null");
  DeviceGuard guard(plan->device);
  free_plan(plan);
  return SAR_OK;
}

}  // extern "C"
