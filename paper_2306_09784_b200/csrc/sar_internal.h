// Internal declarations shared by the libsar translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>

#include "../../include/sar_bp.h"

namespace sar {

constexpr double kLightSpeed = 299792458.0;  // m/s
constexpr double kPi = 3.14159265358979323846;

// BP pixel tile of one CTA: 32 x (ncw * pb) pixels (see bp_kernel.cu for the
// warp/lane -> pixel map).
constexpr int kTileX = 32;
constexpr int kBpMaxStages = 8;          // shared-memory ring depth limit
constexpr int kMaxDevices = 64;          // per-device launch configuration caches

// Range-compression kernel arguments (rc_kernel.cu).
struct RcArgs {
  const float* raw;        // [rows][ns], row = m * n_rx + n
  const float* wsar;       // [n_chirps] or nullptr
  const float* window;     // [ns] range window (plan table)
  const float2* twiddle;   // [nfft/2] exp(-j 2 pi q / nfft) (plan table)
  const float2* ramp;      // [n_bins] exp(+j 2 pi k t_c / nfft), k = k_lo + i (plan table)
  float2* prof;            // [rows][n_bins]
  int row0, nrows;         // rows of the chirp shard
  int n_rx, ns, nfft, log2n, k_lo, n_bins;
  float scale;             // 2 / sum(window)
  // register path (rc_path() = L > 0): plan tables built in fp64
  const float2* coef;      // [N/L][ns]  w[t] exp(-j 2 pi b t / N): window x stage-0 pre-twiddle
  const float2* stw;       // stage twiddles: [8][8] W_64^(k r), then [64][R2] W_L^(k r)
};

// Back-projection kernel arguments (bp_kernel.cu).
struct BpArgs {
  const float2* prof;      // [n_chirps][n_rx][n_bins]
  const double* tx;        // [n_chirps][3]
  const double* rx;        // [n_chirps][n_rx][3] or nullptr (monostatic)
  const float* dop;        // [ny][nx] or nullptr
  const float2* binphase;  // [n_bins+1] exp(j 2 pi beta (k_lo + k + 1/2)), k = -1.., beta = c2/a1
  float2* img;             // [nrow][nx]
  // image rows [row0, row0 + nrow) of the grid (img points at row row0).  A launch covers the
  // whole tile rows [ty0, ty0 + ntile / tiles_x) (launch-local tile t = (ty - ty0) * tiles_x + tx);
  // the CTAs compute the tiles t in [tile_lo, tile_hi) and store only their pixels inside the rows
  int n_bins, n_rx, chirp0, nchirp, row0, nrow, nx, tiles_x, accumulate;
  int ty0, ntile, tile_lo, tile_hi;
  int ksplit, chunk;        // chirp split (launcher): ksplit chunks of `chunk` chirps
  int W;                   // window bins per item
  float dop_max;           // declared |f_doppler| bound (bins): the table is clamped to it
  int derive;              // 1: derived-chirp groups allowed (monostatic far-field tiles)
  int CB;                  // chirps per ring stage
  int S;                   // ring stages (<= kBpMaxStages)
  int ncw, pb;             // CTA shape: consumer warps, pixels per consumer thread
  double x0, y0, z0, dx, dy;
  int polar;               // 0: Cartesian (x0, y0, z0, dx, dy); 1: polar, centre (x0, y0, z0)
  double r0, dr, th0, dth; // polar grid (Measure E)
  double a1, c2, k_lo;     // bins / metre two-way, cycles / metre two-way, crop start
  double kap_half;         // half window span in bins: 2 a1 rho_win + doppler bound
  double box_lo[3], box_hi[3];  // declared antenna box (near-field tile test)
  double tile_rho;         // Cartesian tile half-diagonal; a tile whose anchor lies within
                           // 3 rho_T + 1 mm of the box runs the SAFE form
  // NEXT-4 scatter epilogue: when n_peer > 0 the tile is stored at absolute rows row0 + j of
  // every full image peer[d] ([ny][nx]; P2P-mapped peer buffers, or one multicast address
  // written with multimem.st when multicast != 0) instead of img
  float2* peer[8];
  int n_peer, multicast;
  // Chirp split: chunk c stores its partial image into plane c of ws ([ws_planes][nrow][nx],
  // plane stride ws_plane elements); the planes are summed in chunk order (deterministic) by the
  // split-sum kernel, or under a scatter by the last chunk of each tile (tile_count, per tile of
  // the launch, zeroed by the launcher), which then stores the finished tile to every peer.
  // ws == nullptr: the launch runs unsplit.
  float2* ws;
  long ws_plane;
  int ws_planes;
  int* tile_count;
  int* split_query;        // non-null: report the chirp chunks of this launch, do not launch
  int* ksplit_out;         // non-null: receives the chirp chunks of the launch
  const float4* pairs;     // pair-format rows [n_chirps * n_rx][pair_stride] (pair_kernel) or nullptr
  int pair_stride, pair_pad;   // entry of crop bin k: k + pair_pad (pad minus the rows' first bin)
  float A1f;               // index slope per metre of Delta-R (2 a1 monostatic, a1 bistatic)
  float C3f;               // 2 pi beta: carrier phase (rad) per range bin
};

bool bp_shape_supported(int ncw, int pb);
size_t bp_smem_bytes(int W, int CB, int n_rx, int S, bool bistatic);
cudaError_t launch_rc(const RcArgs& a, cudaStream_t s);
int rc_path(int ns, int nfft, bool allow_env = true);   // 0: classic shared-memory FFT, else the register path's L
cudaError_t launch_bp(const BpArgs& a, bool bistatic, bool doppler, bool near, cudaStream_t s);
cudaError_t launch_bp_scatter(const BpArgs& a, bool bistatic, bool doppler, bool near, cudaStream_t s);

// Doppler-table kernel arguments (doppler_kernel.cu).
struct DopArgs {
  float* out;              // [ny][nx]
  double x0, y0, z0, dx, dy;
  int nx, ny;
  int polar;               // 1: polar grid, centre (x0, y0, z0), (r0, dr, th0, dth); nx = n_th, ny = n_r
  double r0, dr, th0, dth;
  double q[3], v[3];       // reference antenna position, average velocity
  double legs;             // 2: TX and RX legs
  double bins_per_mps;     // f0 / c / (fs / N): bins per m/s of radial speed
};
cudaError_t launch_doppler(const DopArgs& a, cudaStream_t s);
cudaError_t launch_sum(float2* out, const float2* in, int n, long stride, long count, cudaStream_t s);
// Chirp-split sum: img[p] = ((img[p] + ws[0][p]) + ws[1][p]) + ... (chunk order; img holds chunk
// 0) for the pixels of the absolute tiles [tile0, tile0 + ntile) inside rows [row0, row0 + nrow)
// (img, ws at row row0).
struct SplitSumArgs {
  float2* img;
  const float2* ws;
  long plane;
  int planes, tile0, ntile, tiles_x, tile_y, row0, nrow, nx;
};
cudaError_t launch_split_sum(const SplitSumArgs& a, cudaStream_t s);
// Publish (SAR_SCATTER_PUBLISH): copy the pixels of the absolute tiles [tile0, tile0 + ntile) of the
// full image src to the same positions of every full image dst[d], d < n_dst.
struct PublishArgs {
  const float2* src;
  float2* dst[8];
  int n_dst, tile0, ntile, tiles_x, tile_y, nx, ny;
};
cudaError_t launch_publish(const PublishArgs& a, cudaStream_t s);

// Polar -> Cartesian resampling arguments (resample_kernel.cu).
struct ResampleArgs {
  const float2* in;        // [n_r][n_th]
  float2* out;             // [ny][nx]
  double xc, yc, r0, dr, th0, dth;
  int n_th, n_r;
  double x0, y0, dx, dy;
  int nx, ny;
};
cudaError_t launch_resample(const ResampleArgs& a, cudaStream_t s);

// Pair-format rows for the BP producer's bulk copies (pair_kernel.cu).
struct PairArgs {
  const float2* prof;      // [rows][n_bins]
  const float2* binphase;  // [n_bins + 1], from k = -1
  float4* out;             // [rows][stride]
  int row0, rows, n_bins, stride, pad;
  int k0;                  // first crop bin the rows cover (a row shard's own crop)
};
cudaError_t launch_pairs(const PairArgs& a, cudaStream_t s);

}  // namespace sar

struct sar_plan_s {
  sar_radar_params_t radar;
  sar_grid_t grid;          // Cartesian grid, or the stand-in (nx = n_th, ny = n_r) of a polar one
  bool polar = false;
  sar_polar_grid_t pgrid{};
  sar_box_t box;
  sar_plan_info_t info;
  int device;
  bool near_field;         // an antenna may come within 2 rho of a tile anchor
  int bp_ncw, bp_pb, bp_stages;
  double tile_rho;         // tile half-diagonal (m), max over tiles
  double win_rho;          // per-leg half spread of |p - q| over a tile (m): sets kap_half
  float rc_scale;
  float* d_window = nullptr;
  float2* d_twiddle = nullptr;
  float2* d_rc_coef = nullptr;   // register-path range-compression tables (rc_kernel.cu)
  float2* d_rc_stw = nullptr;
  float2* d_ramp = nullptr;
  float2* d_binphase = nullptr;
  // sar_form_image workspace (lazily allocated under ws_mutex)
  std::mutex ws_mutex;
  float* w_raw = nullptr;
  float* w_wsar = nullptr;
  double* w_tx = nullptr;
  double* w_rx = nullptr;
  float* w_dop = nullptr;
  float2* w_prof = nullptr;
  float2* w_img = nullptr;
  cudaStream_t w_copy = nullptr;   // sar_form_image: readback stream of the banded pipeline
  cudaEvent_t w_ev[9] = {};        // band-done events (8 bands max) + the last copy's
  cudaMemPool_t pool = nullptr;   // device pool of the per-call pair-format rows (not owned)
  std::atomic<int64_t> launches{0};
};
