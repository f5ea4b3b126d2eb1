/*
 * sar_bp.h -- C ABI of the B200-native FMCW range compression + time-domain
 * Back-Projection (BP) library (libsar.so), arXiv 2306.09784.
 *
 * Citations: "P:Lnnn" is a line of the paper text; A1..A17 are the
 * readings of the paper listed in DESIGN.md.
 *
 * Conventions for every entry point
 *   - Plain C types only.  "dev" pointers are CUDA device pointers on the plan's
 *     device; "host" pointers are host memory (pinned memory makes the copies of
 *     sar_form_image asynchronous).  Complex numbers are interleaved (re, im)
 *     float32 pairs (sar_complex64_t), the layout of torch.complex64.
 *   - Ownership: the caller owns every buffer it passes.  The plan owns only its
 *     constant tables (range window, FFT twiddles, centring ramp) and, once
 *     sar_form_image is used, a device workspace; sar_destroy frees them.
 *   - Streams: sar_stream_t is a cudaStream_t (NULL = legacy default stream).
 *     Every call is stream-ordered and asynchronous; argument errors are returned
 *     before anything is enqueued.  Asynchronous device faults surface at the
 *     caller's next synchronisation as CUDA errors.
 *   - Errors: every call returns a sar_status_t and never throws across the ABI;
 *     sar_last_error() gives a thread-local message for the last failure.
 *   - The plan is immutable after creation: concurrent calls on different streams
 *     with disjoint output buffers are allowed -- except sar_form_image, whose
 *     device workspace belongs to the plan: its calls on one plan must share one
 *     stream (or be serialised by the caller).
 */
#ifndef SAR_BP_H
#define SAR_BP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sar_plan_s* sar_plan_t;
typedef void* sar_stream_t; /* cudaStream_t */

typedef struct {
  float re, im;
} sar_complex64_t;

typedef enum {
  SAR_OK = 0,
  SAR_ERR_INVALID_ARGUMENT = 1,  /* null pointer, violated invariant, shard out of range */
  SAR_ERR_OUT_OF_COVERAGE = 2,   /* an antenna position lies outside the declared box */
  SAR_ERR_CUDA = 3,              /* a CUDA runtime call failed */
  SAR_ERR_NO_MEMORY = 4,         /* host or device allocation failed */
  SAR_ERR_UNSUPPORTED_DEVICE = 5 /* device is not an sm_100 (B200-class) GPU */
} sar_status_t;

/* Radar and waveform parameters: Table 1 plus the quantities the
 * paper does not give (A5, A6).  Invariants checked by sar_plan_create:
 * all times/frequencies > 0, pri_s >= chirp_s, n_samples >= 2,
 * round(sample_rate_hz * chirp_s) == n_samples, fft_len a power of two with
 * n_samples <= fft_len <= 16384, n_chirps >= 1, n_rx >= 1, range_window in {0,1},
 * doppler_max_bins >= 0. */
typedef struct {
  double f0_hz;            /* carrier: instantaneous frequency at the chirp centre (A4) */
  double bandwidth_hz;     /* B; chirp rate mu = B / T_P */
  double chirp_s;          /* T_P */
  double pri_s;            /* T_P0; informational (real-time budget P:L217) */
  double sample_rate_hz;   /* fs of the real ADC samples (A5, A7) */
  int32_t n_samples;       /* Ns, real samples per chirp */
  int32_t n_chirps;        /* capacity M: profiles/poses arrays hold M chirps */
  int32_t n_rx;            /* receive channels per chirp (one TX) */
  int32_t fft_len;         /* N_fft: zero-padded FFT length (Z = N_fft / Ns, A6) */
  int32_t range_window;    /* 0 rectangular, 1 symmetric Hann (A6) */
  float doppler_max_bins;  /* declared bound on |f_doppler(p)| in bins (Alg. 2 L8,
                              P:L470); 0 when sar_backproject gets no Doppler array */
} sar_radar_params_t;

/* Cartesian pixel grid in the plane z = z0: pixel (i, j) is at
 * (x0 + i dx, y0 + j dy, z0), i in [0, nx), j in [0, ny) (A12, A13).
 * Images are row-major [ny][nx] (x fastest).  dx, dy > 0; nx, ny >= 1. */
typedef struct {
  double x0, y0, z0, dx, dy;
  int32_t nx, ny;
} sar_grid_t;

/* Polar reconstruction grid of Measure E: "a new grid ... that originates in
 * the center of the synthetic aperture", range and azimuth spacing a factor finer than the
 * PSF resolutions.  Pixel (i, j), i in [0, n_th) (bearing, fastest), j in [0, n_r) (range):
 *   r_j = r0 + j dr,  th_i = th0 + i dth (radians from +y toward +x),
 *   p = (xc + r_j sin th_i, yc + r_j cos th_i, zc).
 * Images are row-major [n_r][n_th].  dr, dth > 0; r0 >= 0; n_th, n_r >= 1. */
typedef struct {
  double xc, yc, zc, r0, dr, th0, dth;
  int32_t n_th, n_r;
} sar_polar_grid_t;

/* Declared axis-aligned bounding box of ALL antenna phase centres (TX and RX)
 * the plan will be used with.  The range crop is derived from it and the grid box
 * with the triangle inequality; positions outside it give wrong values (never an
 * out-of-bounds access: pair-row copies are clamped into their row, and a polar plan,
 * whose tile windows are bounded with the box, clamps positions into the box).
 * sar_form_image verifies its host positions against it. */
typedef struct {
  double lo[3], hi[3];
} sar_box_t;

/* Derived plan quantities (host-side maths, no device needed). */
typedef struct {
  double chirp_rate_hz_per_s; /* mu = B / T_P */
  double a1_bins_per_m;       /* f_ind = a1 * d_hyp: mu N_fft / (c fs) per metre of
                                 two-way path (Alg. 2 L8; A6) */
  double c2_cycles_per_m;     /* s_hyp = exp(j 2 pi c2 d_hyp), c2 = f0 / c (Alg. 2 L9,
                                 P:L472; A2, A3) */
  double d_min_m, d_max_m;    /* bounds of d_hyp over grid x antenna box */
  int32_t k_lo;               /* first profile bin kept by the crop */
  int32_t n_bins;             /* profile row length (bins k_lo .. k_lo+n_bins-1) */
  int32_t tile_x, tile_y;     /* BP pixel tile of one CTA */
  int32_t window_bins;        /* profile bins staged per (tile, chirp, rx) */
  int32_t chirps_per_stage;   /* chirps per shared-memory ring stage */
  int64_t updates_per_image;  /* nx * ny * n_chirps * n_rx */
  double window_half_bins;    /* bound on |kappa(p) - kappa(anchor)| over a tile (bins,
                                 incl. the Doppler bound); the staged window is
                                 [floor(kappa_anchor - half) - 1, + window_bins) */
  double tile_rho_m;          /* largest tile half-diagonal (m) */
} sar_plan_info_t;

/* Validate parameters and compute the derived quantities without touching a GPU.
 * Returns SAR_ERR_INVALID_ARGUMENT on a violated invariant. */
sar_status_t sar_plan_geometry(const sar_radar_params_t* radar, const sar_grid_t* grid,
                               const sar_box_t* antenna_box, sar_plan_info_t* info);

/* Create a plan on CUDA device `device`: validates as sar_plan_geometry, checks the
 * device is sm_100 (else SAR_ERR_UNSUPPORTED_DEVICE), builds the range window,
 * FFT twiddle and centring-ramp tables in double, rounds them to float32 and
 * uploads them (synchronously, once).  *out receives the plan. */
sar_status_t sar_plan_create(const sar_radar_params_t* radar, const sar_grid_t* grid,
                             const sar_box_t* antenna_box, int32_t device, sar_plan_t* out);

/* Polar-grid plan (Measure E): as sar_plan_create, for a sar_polar_grid_t.  All other calls
 * work unchanged on it, with "rows" = range rings j and "nx" = n_th bearings. */
sar_status_t sar_plan_create_polar(const sar_radar_params_t* radar, const sar_polar_grid_t* grid,
                                   const sar_box_t* antenna_box, int32_t device, sar_plan_t* out);
sar_status_t sar_plan_geometry_polar(const sar_radar_params_t* radar, const sar_polar_grid_t* grid,
                                     const sar_box_t* antenna_box, sar_plan_info_t* info);

/* Resample a polar image onto a Cartesian grid "for comparability": bilinear
 * interpolation of the complex values in (th, r) for each Cartesian pixel centre; pixels
 * outside the polar coverage are 0.
 *   polar_image dev complex [n_r][n_th] of `polar`; out dev complex [ny][nx] of `cart`. */
sar_status_t sar_polar_to_cartesian(const sar_polar_grid_t* polar, const sar_complex64_t* polar_image,
                                    const sar_grid_t* cart, sar_complex64_t* out, sar_stream_t stream);

sar_status_t sar_plan_info(sar_plan_t plan, sar_plan_info_t* info);

/* Profile row geometry: bins k_lo .. k_lo + n_bins - 1 of the one-sided
 * zero-padded spectrum are kept (range-bin cropping, north star). */
sar_status_t sar_plan_crop(sar_plan_t plan, int32_t* k_lo, int32_t* n_bins);

/* Range compression (step H1; A4-A8).  For every chirp m in
 * [chirp0, chirp0 + nchirp) and RX n:
 *   X[k] = (2 w_sar[m] / sum_t w[t]) sum_{t<Ns} w[t] raw[m][n][t] exp(-j 2 pi k (t - t_c) / N_fft)
 * for k in the crop, t_c = (Ns - 1) / 2, w the range window.  Batched pruned
 * real-to-complex FFT: only the cropped bins are written.
 *   raw       dev float   [n_chirps][n_rx][n_samples]   (read: chirps of the shard)
 *   w_sar     dev float   [n_chirps] per-chirp aperture window (Measure B,
 *                         P:L298-299), or NULL for w_sar = 1
 *   profiles  dev complex [n_chirps][n_rx][n_bins]      (written: chirps of the shard)
 * 0 <= chirp0, 0 <= nchirp, chirp0 + nchirp <= n_chirps; nchirp == 0 is a no-op. */
sar_status_t sar_range_compress(sar_plan_t plan, const float* raw, const float* w_sar,
                                int32_t chirp0, int32_t nchirp, sar_complex64_t* profiles,
                                sar_stream_t stream);

/* Back-Projection (steps H2-H6; Alg. 2): for every pixel p of rows
 * [row0, row0 + nrow) and every chirp m of [chirp0, chirp0 + nchirp):
 *   P(p) (+)= sum_m sum_n s(a1 d_hyp + f_doppler(p), m, n) exp(+j 2 pi c2 d_hyp)
 *   d_hyp = |p - q_tx(m)| + |p - q_rx(m, n)|,  s(kappa) linear interpolation of the
 *   profile row (A8, A9), zero outside the one-sided spectrum.
 *   profiles  dev complex [n_chirps][n_rx][n_bins] from sar_range_compress
 *   tx_pos    dev double  [n_chirps][3] TX phase centres (any order, any track)
 *   rx_pos    dev double  [n_chirps][n_rx][3] RX phase centres, or NULL for
 *                         monostatic q_rx = q_tx (then n_rx must be 1)
 *   doppler_bins dev float [ny][nx] per-pixel f_doppler in bins (Measure D,
 *                         P:L311-317) or NULL (no Doppler term, A10); requires
 *                         doppler_max_bins >= max |doppler_bins| in the plan (values
 *                         beyond it are clamped to +-doppler_max_bins)
 *   image     dev complex [nrow][nx]: row r holds grid row row0 + r
 *   accumulate 0: image = P;  1: image += P (chirp sharding, NCCL reduce)
 * nrow == 0 is a no-op; nchirp == 0 writes zeros (accumulate = 0) or nothing.
 * Pixels are computed in absolute grid tiles (see sar_backproject_tiles), so any row shard
 * reproduces the unsharded image's pixels.  A launch too small to fill the GPU splits its
 * chirps into chunks whose partial images (stream-ordered workspace from the plan's pool) are
 * summed in chunk order by a second kernel: results are bit-reproducible run to run. */
sar_status_t sar_backproject(sar_plan_t plan, const sar_complex64_t* profiles,
                             const double* tx_pos, const double* rx_pos,
                             const float* doppler_bins, int32_t chirp0, int32_t nchirp,
                             int32_t row0, int32_t nrow, sar_complex64_t* image,
                             int32_t accumulate, sar_stream_t stream);

/* Back-projection with the image gather (or the chirp-shard reduction) fused into the
 * epilogue (NEXT-4; the north star's multi-GPU design): the same computation as
 * sar_backproject for rows [row0, row0 + nrow) and chirps [chirp0, chirp0 + nchirp), but every
 * finished tile goes to its ABSOLUTE rows row0 + j of each full image images[d] (complex
 * [ny][nx], d < n_images <= 8) while the remaining tiles are still being computed:
 *   flags = 0                   store (pixel-row shards: the gather)
 *   flags |= SAR_SCATTER_ADD    atomic add (chirp shards: the reduction; images must hold the
 *                               running sum, e.g. zeroed before the first shard)
 *   flags |= SAR_SCATTER_MULTICAST  images[0] is an NVSwitch multicast address (n_images = 1):
 *                               multimem.st / multimem.red reach every rank's image at once
 * With symmetric memory the images are the P2P-mapped buffers of every rank (one NVLink
 * store or reduction per peer).  Rows outside [row0, row0 + nrow) are not touched; the caller
 * orders the ranks (e.g. a symmetric-memory barrier) before reading.  A store scatter runs
 * chirp-split (to about 16 waves of resident CTAs): each chunk stores its partial
 * tile into its own plane of a stream-ordered workspace from the plan's pool and the last chunk
 * of each tile sums the planes in chunk order and stores the finished tile (SAR_ERR_NO_MEMORY
 * never results: without the workspace it runs unsplit).  SAR_SCATTER_ADD runs unsplit; its
 * cross-rank additions land in arrival order (fp32: not bit-reproducible across runs).
 *   images  host array of n_images device pointers (may be peer or multicast addresses) */
#define SAR_SCATTER_MULTICAST 1
#define SAR_SCATTER_ADD 2
/* sar_backproject_scatter_tiles only: compute first, then publish.  images[0] is the caller's OWN
 * full image: the tiles are back-projected into it exactly as by sar_backproject_tiles (plain
 * kernels, chirp chunks summed by the split-sum kernel), then one copy kernel stores the finished
 * tiles at their absolute positions of images[1..n_images) (P2P stores over NVLink).  The copy
 * does not overlap the compute but costs about one pass over the rank's pixels per peer, while
 * the fused epilogue's split publish measured 4.5-6 % more BP time per rank (round 2).  Not with
 * SAR_SCATTER_ADD or SAR_SCATTER_MULTICAST. */
#define SAR_SCATTER_PUBLISH 4
sar_status_t sar_backproject_scatter(sar_plan_t plan, const sar_complex64_t* profiles,
                                     const double* tx_pos, const double* rx_pos,
                                     const float* doppler_bins, int32_t chirp0, int32_t nchirp,
                                     int32_t row0, int32_t nrow, sar_complex64_t* const* images,
                                     int32_t n_images, int32_t flags, sar_stream_t stream);

/* Tile shards ("rank r owns a contiguous block of tiles"; T11).  The BP computes
 * the grid in absolute tiles of tile_x x tile_y pixels (sar_plan_info), tile t = ty * tiles_x + tx
 * covering columns [tx tile_x, +tile_x) and rows [ty tile_y, +tile_y) clipped to the grid, each
 * with its own fp64 anchor at the tile centre.  Every pixel is therefore computed identically by
 * any row shard, tile shard or unsharded call that contains it (pixel independence of Alg. 2,
 * P:L459); images differ only in the fp32 order of chirp-chunk sums when the launches
 * split their chirps differently (<= 1e-6 relative).
 *
 * sar_plan_tiles: tiles_x = ceil(nx / tile_x), tiles_y = ceil(ny / tile_y). */
sar_status_t sar_plan_tiles(sar_plan_t plan, int32_t* tiles_x, int32_t* tiles_y);

/* sar_backproject over the absolute tiles [tile0, tile0 + ntile) (0 <= tile0, tile0 + ntile <=
 * tiles_x * tiles_y; ntile == 0 is a no-op) for chirps [chirp0, chirp0 + nchirp):
 *   image  dev complex [ny][nx], the FULL image (absolute rows): only the pixels of the tiles
 *          in range are written (accumulate 0: =, 1: +=); all other pixels are untouched.
 * Errors as sar_backproject. */
sar_status_t sar_backproject_tiles(sar_plan_t plan, const sar_complex64_t* profiles, const double* tx_pos,
                                   const double* rx_pos, const float* doppler_bins, int32_t chirp0,
                                   int32_t nchirp, int32_t tile0, int32_t ntile, sar_complex64_t* image,
                                   int32_t accumulate, sar_stream_t stream);

/* sar_backproject_scatter over the absolute tiles [tile0, tile0 + ntile): every finished tile is
 * stored (or added, SAR_SCATTER_ADD) at its absolute position of each full image images[d]. */
sar_status_t sar_backproject_scatter_tiles(sar_plan_t plan, const sar_complex64_t* profiles,
                                           const double* tx_pos, const double* rx_pos,
                                           const float* doppler_bins, int32_t chirp0, int32_t nchirp,
                                           int32_t tile0, int32_t ntile, sar_complex64_t* const* images,
                                           int32_t n_images, int32_t flags, sar_stream_t stream);

/* End-to-end image formation from HOST buffers (the paper's "Load" + "BP",
 * Table 2, pinned memory P:L357-360): copies raw, w_sar and poses to a
 * plan-owned device workspace, runs sar_range_compress over all chirps and
 * sar_backproject over all chirps for grid rows [row0, row0 + nrow), and returns
 * those image rows, all on `stream`.  When image_host is pinned (device-mapped), the rows
 * run as up to 4 bands of whole tile rows and each band is copied to image_host (on a
 * plan-owned copy stream) while the next band computes -- the readback overlapped with the
 * compute; a single tile row instead has the BP epilogue store each finished tile straight
 * into image_host.  Otherwise one copy follows the kernel.  A pinned raw_host is read by the range
 * compression directly.
 *   raw_host [n_chirps][n_rx][n_samples] float; w_sar_host [n_chirps] float or NULL;
 *   tx_host [n_chirps][3] double; rx_host [n_chirps][n_rx][3] double or NULL;
 *   doppler_host [ny][nx] float or NULL; image_host [nrow][nx] complex (written).
 * Positions are checked against the declared antenna box first
 * (SAR_ERR_OUT_OF_COVERAGE).  The caller synchronises `stream` before reading
 * image_host. */
sar_status_t sar_form_image(sar_plan_t plan, const float* raw_host, const float* w_sar_host,
                            const double* tx_host, const double* rx_host,
                            const float* doppler_host, int32_t row0, int32_t nrow,
                            sar_complex64_t* image_host, sar_stream_t stream);

/* Per-pixel Doppler index shift of Measure D (Alg. 2 L8 f_doppler(p)): "the
 * radial component for every pixel p can be calculated in advance based on the average
 * vehicle velocity".  For pixel p of `grid`:
 *   v_r(p) = n_legs <p - q_ref, v_avg> / |p - q_ref|     (TX and RX legs, n_legs = 2)
 *   f_doppler(p) = (f0 v_r(p) / c) / (fs / N_fft)        in profile bins,
 * with q_ref the aperture-centre antenna position and v_avg the average velocity (host,
 * metres and m/s).  |f_doppler| <= 2 f0 |v_avg| N_fft / (c fs): declare that bound (or the
 * table's max) as doppler_max_bins in the plan that consumes the table.
 *   doppler_bins  dev float [ny][nx] (written); a pixel at q_ref gets 0.
 * Computed on `stream` in fp64, stored as float32.  No plan needed. */
sar_status_t sar_doppler_table(const sar_radar_params_t* radar, const sar_grid_t* grid,
                               const double q_ref[3], const double v_avg[3], float* doppler_bins,
                               sar_stream_t stream);

/* The same table for the pixels of a Measure E polar grid (image layout [n_r][n_th]). */
sar_status_t sar_doppler_table_polar(const sar_radar_params_t* radar, const sar_polar_grid_t* grid,
                                     const double q_ref[3], const double v_avg[3], float* doppler_bins,
                                     sar_stream_t stream);

/* Incremental streaming (NEXT-2; continuous processing): with a
 * world-fixed grid, a frame over an aperture of n_partials hops is the sum of the hops'
 * partial images (each sar_backproject over one hop of chirps).  Writes
 *   out[i] = sum_{k < n_partials} partials[k * stride + i],  i < n_elems
 * summed in k order (deterministic).  partials: dev complex ring [n_partials][stride];
 * out: dev complex [n_elems].  n_partials >= 1, stride >= n_elems. */
sar_status_t sar_image_sum(sar_complex64_t* out, const sar_complex64_t* partials, int32_t n_partials,
                           int64_t stride, int64_t n_elems, sar_stream_t stream);

/* Number of CUDA kernels this plan has launched since creation. */
int64_t sar_plan_launch_count(sar_plan_t plan);

/* Release the plan's tables and workspace (after pending work on them finished). */
sar_status_t sar_destroy(sar_plan_t plan);

/* Thread-local message describing the last non-OK status on this thread. */
const char* sar_last_error(void);

/* Library version string. */
const char* sar_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SAR_BP_H */
