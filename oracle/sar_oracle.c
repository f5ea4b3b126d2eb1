/*
 * oracle/sar_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, double-precision CPU oracle for the hot path of arXiv 2306.09784
 * ("Implementation of Real-Time Automotive SAR Imaging"): FMCW range compression
 * followed by time-domain Back-Projection (BP).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load this library.  It shares no code, header, table or
 * constant with the CUDA path under paper_2306_09784_b200/.
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn; readings A1..A17 are
 * listed in DESIGN.md ("Readings of the paper").
 *
 * Every function here is pinned by a -m "not gpu" test against something other
 * than itself (see tests/test_oracle_pins.py).  Parity status per function:
 *   oracle_window          pinned (numpy.hanning; closed-form endpoints)
 *   oracle_dft_row         pinned (exact-bin tone closed form, numpy.fft.rfft)
 *   oracle_fft             pinned (literal DFT, numpy.fft.fft, Parseval)
 *   oracle_range_compress  pinned (literal DFT, exact-bin tone, zero input)
 *   oracle_backproject     pinned (flat-profile closed form, exact-bin circular
 *                          track, point-target argmax and phase, permutation,
 *                          translation, linearity, brute-force numpy on tiny input)
 *   oracle_polar_to_cartesian  pinned (node values reproduced, functions bilinear in
 *                          (th, r) reproduced exactly, constant image, outside = 0)
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define ORACLE_C_LIGHT 299792458.0 /* m/s, exact (SI definition) */
#define ORACLE_PI 3.14159265358979323846

int oracle_version(void) { return 1; }

/* Range window over fast time.  kind 0: rectangular (w = 1).  kind 1: symmetric
 * Hann w[t] = 0.5 - 0.5 cos(2 pi t / (Ns - 1)), t = 0..Ns-1 (reading A6; the north
 * star asks for "windowing" without naming the family). */
int oracle_window(int ns, int kind, double* w) {
  if (ns < 1 || !w) return -1;
  for (int t = 0; t < ns; ++t) {
    if (kind == 0 || ns == 1)
      w[t] = 1.0;
    else if (kind == 1)
      w[t] = 0.5 - 0.5 * cos(2.0 * ORACLE_PI * (double)t / (double)(ns - 1));
    else
      return -1;
  }
  return 0;
}

/* Literal range-compression sum for one beat row (reading A7, C-1 step 2):
 *   X[k] = scale * sum_{t=0}^{Ns-1} w[t] x[t] exp(-j 2 pi k (t - t_c) / N),
 *   t_c = (Ns - 1)/2, for 0 <= k <= N/2, and X[k] = 0 outside [0, N/2] (A8).
 * Output bins k = k0 .. k0+nk-1, interleaved (re, im).  O(Ns * nk). */
int oracle_dft_row(const double* x, int ns, int nfft, const double* w, double scale,
                   int k0, int nk, double* out) {
  if (!x || !w || !out || ns < 1 || nfft < ns || nk < 0) return -1;
  const double tc = 0.5 * (double)(ns - 1);
  for (int i = 0; i < nk; ++i) {
    const int k = k0 + i;
    double re = 0.0, im = 0.0;
    if (k >= 0 && k <= nfft / 2) {
      for (int t = 0; t < ns; ++t) {
        const double arg = -2.0 * ORACLE_PI * (double)k * ((double)t - tc) / (double)nfft;
        re += w[t] * x[t] * cos(arg);
        im += w[t] * x[t] * sin(arg);
      }
    }
    out[2 * i] = scale * re;
    out[2 * i + 1] = scale * im;
  }
  return 0;
}

/* Textbook iterative radix-2 decimation-in-time forward FFT, in place:
 *   Z[k] = sum_t z[t] exp(-j 2 pi k t / n),  n a power of two.
 * (bit-reversal permutation, then log2(n) butterfly passes; twiddles from a
 * cos/sin table of exp(-j 2 pi q / n), q < n/2). */
int oracle_fft(double* re, double* im, int n) {
  if (!re || !im || n < 1 || (n & (n - 1))) return -1;
  if (n == 1) return 0;
  for (int i = 1, j = 0; i < n; ++i) { /* bit reversal */
    int bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      double tr = re[i]; re[i] = re[j]; re[j] = tr;
      double ti = im[i]; im[i] = im[j]; im[j] = ti;
    }
  }
  double* cw = (double*)malloc(sizeof(double) * (size_t)(n / 2));
  double* sw = (double*)malloc(sizeof(double) * (size_t)(n / 2));
  if (!cw || !sw) { free(cw); free(sw); return -2; }
  for (int q = 0; q < n / 2; ++q) {
    cw[q] = cos(-2.0 * ORACLE_PI * (double)q / (double)n);
    sw[q] = sin(-2.0 * ORACLE_PI * (double)q / (double)n);
  }
  for (int len = 2; len <= n; len <<= 1) {
    const int half = len / 2, stride = n / len;
    for (int s = 0; s < n; s += len) {
      for (int j = 0; j < half; ++j) {
        const double wr = cw[j * stride], wi = sw[j * stride];
        const int a = s + j, b = s + j + half;
        const double br = re[b] * wr - im[b] * wi;
        const double bi = re[b] * wi + im[b] * wr;
        re[b] = re[a] - br; im[b] = im[a] - bi;
        re[a] = re[a] + br; im[a] = im[a] + bi;
      }
    }
  }
  free(cw); free(sw);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Range compression (step H1; "equidistantly spaced" beat  */
/* frequency axis; readings A5-A8).  raw: float32 [n_chirps][n_rx][ns] real    */
/* beat samples.  wsar: per-chirp aperture window w_sar(m) or NULL */
/* (= 1).  For every row (m, n):                                               */
/*   X[k] = (2 w_sar[m] / sum_t w[t]) * sum_t w[t] x[t] exp(-j2pi k (t-t_c)/N)  */
/* computed as the forward FFT of the zero-padded windowed row times the        */
/* centring ramp exp(+j 2 pi k t_c / N) (use_dft = 0), or literally            */
/* (use_dft = 1).  Output bins k0..k0+nk-1 (zero outside [0, N/2]):            */
/* out [n_chirps][n_rx][nk][2] doubles.                                         */
/* ------------------------------------------------------------------------- */
typedef struct {
  const float* raw; const double* wsar; const double* w; double wsum;
  int n_chirps, n_rx, ns, nfft, k0, nk, use_dft;
  double* out; int row_begin, row_end; int status;
} rc_job_t;

static void* rc_worker(void* arg) {
  rc_job_t* j = (rc_job_t*)arg;
  const int n = j->nfft;
  double* re = (double*)malloc(sizeof(double) * (size_t)n);
  double* im = (double*)malloc(sizeof(double) * (size_t)n);
  double* x = (double*)malloc(sizeof(double) * (size_t)j->ns);
  if (!re || !im || !x) { j->status = -2; free(re); free(im); free(x); return NULL; }
  const double tc = 0.5 * (double)(j->ns - 1);
  for (int row = j->row_begin; row < j->row_end; ++row) {
    const int m = row / j->n_rx;
    const double scale = 2.0 * (j->wsar ? j->wsar[m] : 1.0) / j->wsum;
    const float* xr = j->raw + (size_t)row * (size_t)j->ns;
    double* o = j->out + (size_t)row * (size_t)j->nk * 2;
    for (int t = 0; t < j->ns; ++t) x[t] = (double)xr[t];
    if (j->use_dft) {
      oracle_dft_row(x, j->ns, n, j->w, scale, j->k0, j->nk, o);
      continue;
    }
    for (int t = 0; t < n; ++t) {
      re[t] = t < j->ns ? j->w[t] * x[t] : 0.0;
      im[t] = 0.0;
    }
    if (oracle_fft(re, im, n)) { j->status = -2; break; }
    for (int i = 0; i < j->nk; ++i) {
      const int k = j->k0 + i;
      double vr = 0.0, vi = 0.0;
      if (k >= 0 && k <= n / 2) {
        const double ang = 2.0 * ORACLE_PI * (double)k * tc / (double)n; /* ramp */
        const double cr = cos(ang), ci = sin(ang);
        vr = scale * (re[k] * cr - im[k] * ci);
        vi = scale * (re[k] * ci + im[k] * cr);
      }
      o[2 * i] = vr;
      o[2 * i + 1] = vi;
    }
  }
  free(re); free(im); free(x);
  return NULL;
}

static int oracle_threads(int nthreads) {
  if (nthreads > 0) return nthreads;
  long p = sysconf(_SC_NPROCESSORS_ONLN);
  return p > 0 ? (int)p : 1;
}

int oracle_range_compress(const float* raw, int n_chirps, int n_rx, int ns, int nfft,
                          int window, const double* wsar, int k0, int nk, int use_dft,
                          int nthreads, double* out) {
  if (!raw || !out || n_chirps < 0 || n_rx < 1 || ns < 1 || nfft < ns || nk < 0)
    return -1;
  if (!use_dft && (nfft & (nfft - 1))) return -1;
  double* w = (double*)malloc(sizeof(double) * (size_t)ns);
  if (!w) return -2;
  if (oracle_window(ns, window, w)) { free(w); return -1; }
  double wsum = 0.0;
  for (int t = 0; t < ns; ++t) wsum += w[t];
  const int rows = n_chirps * n_rx;
  int nt = oracle_threads(nthreads);
  if (nt > rows) nt = rows > 0 ? rows : 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nt);
  rc_job_t* jobs = (rc_job_t*)malloc(sizeof(rc_job_t) * (size_t)nt);
  if (!th || !jobs) { free(w); free(th); free(jobs); return -2; }
  for (int i = 0; i < nt; ++i) {
    rc_job_t jb = {raw, wsar, w, wsum, n_chirps, n_rx, ns, nfft, k0, nk, use_dft, out,
                   (int)((long)rows * i / nt), (int)((long)rows * (i + 1) / nt), 0};
    jobs[i] = jb;
    pthread_create(&th[i], NULL, rc_worker, &jobs[i]);
  }
  int status = 0;
  for (int i = 0; i < nt; ++i) {
    pthread_join(th[i], NULL);
    if (jobs[i].status) status = jobs[i].status;
  }
  free(w); free(th); free(jobs);
  return status;
}

/* ------------------------------------------------------------------------- */
/* Back-Projection (steps H3-H5), the plain definition of Alg. 2   */
/* with the constants of Alg. 1 written out:                       */
/*   for every pixel p, for every chirp m (outer), for every RX n (inner):      */
/*     d_tx  = || p - q_tx(m) ||_2                       Alg.2 L4    */
/*     d_rx  = || p - q_rx(m,n) ||_2                     Alg.2 L6    */
/*     d_hyp = d_tx + d_rx                                Alg.2 L7    */
/*     tau   = d_hyp / c                                  Alg.1 L10    */
/*     f_ind = (mu tau) / (fs/N) + f_doppler(p)           Alg.2 L8, Alg.1 L11   */
/*     s_hyp = exp(+j 2 pi f0 tau)                        Alg.2 L9 (A2, A3)     */
/*     P(p) += s_hyp * s(f_ind, m, n)                     Alg.2 L10, L12        */
/*   s(kappa) = (1-f) X[k] + f X[k+1], k = floor(kappa), f = kappa - k (A8, A9), */
/*   X zero outside [0, N/2].  w_sar is already inside X (folded by           */
/*   oracle_range_compress, Measure B P:L298-299).  mu = B/T_P.        */
/* prof: [n_chirps][n_rx][nk][2] doubles holding bins k0..k0+nk-1.  If a pixel  */
/* needs a bin in [0, N/2] that the given crop does not hold, return -3.       */
/* rx == NULL: monostatic, q_rx(m,0) = q_tx(m) (n_rx must be 1).               */
/* ------------------------------------------------------------------------- */
typedef struct {
  const double* prof; int n_chirps, n_rx, k0, nk;
  double f0, mu, fs, nfft;
  const double* tx; const double* rx; const double* dop; const double* pix;
  double* out; int p_begin, p_end; int status;
} bp_job_t;

static int fetch_bin(const bp_job_t* j, const double* row, long k, double* vr, double* vi) {
  *vr = 0.0; *vi = 0.0;
  if (k < 0 || k > (long)(j->nfft / 2)) return 0; /* zero extension (A8) */
  if (k < j->k0 || k >= (long)j->k0 + j->nk) return -3; /* crop too small */
  *vr = row[2 * (k - j->k0)];
  *vi = row[2 * (k - j->k0) + 1];
  return 0;
}

static void* bp_worker(void* arg) {
  bp_job_t* j = (bp_job_t*)arg;
  for (int p = j->p_begin; p < j->p_end; ++p) {
    const double px = j->pix[3 * p], py = j->pix[3 * p + 1], pz = j->pix[3 * p + 2];
    double acc_re = 0.0, acc_im = 0.0;
    for (int m = 0; m < j->n_chirps; ++m) {
      const double* qt = j->tx + 3 * (size_t)m;
      const double d_tx = sqrt((px - qt[0]) * (px - qt[0]) + (py - qt[1]) * (py - qt[1]) +
                               (pz - qt[2]) * (pz - qt[2]));
      for (int n = 0; n < j->n_rx; ++n) {
        double d_rx;
        if (j->rx) {
          const double* qr = j->rx + 3 * ((size_t)m * (size_t)j->n_rx + (size_t)n);
          d_rx = sqrt((px - qr[0]) * (px - qr[0]) + (py - qr[1]) * (py - qr[1]) +
                      (pz - qr[2]) * (pz - qr[2]));
        } else {
          d_rx = d_tx;
        }
        const double d_hyp = d_tx + d_rx;
        const double tau = d_hyp / ORACLE_C_LIGHT;
        double f_ind = (j->mu * tau) / (j->fs / j->nfft);
        if (j->dop) f_ind += j->dop[p];
        const double kf = floor(f_ind);
        const double f = f_ind - kf;
        const double* row = j->prof + ((size_t)m * (size_t)j->n_rx + (size_t)n) * (size_t)j->nk * 2;
        double x0r, x0i, x1r, x1i;
        if (fetch_bin(j, row, (long)kf, &x0r, &x0i) || fetch_bin(j, row, (long)kf + 1, &x1r, &x1i)) {
          j->status = -3;
          return NULL;
        }
        const double sr = (1.0 - f) * x0r + f * x1r;
        const double si = (1.0 - f) * x0i + f * x1i;
        const double ph = 2.0 * ORACLE_PI * j->f0 * tau;
        const double hr = cos(ph), hi = sin(ph);
        acc_re += hr * sr - hi * si;
        acc_im += hr * si + hi * sr;
      }
    }
    j->out[2 * p] = acc_re;
    j->out[2 * p + 1] = acc_im;
  }
  return NULL;
}

int oracle_backproject(const double* prof, int n_chirps, int n_rx, int k0, int nk,
                       double f0_hz, double bandwidth_hz, double chirp_s, double fs_hz,
                       int nfft, const double* tx, const double* rx, const double* doppler,
                       const double* pix, int n_pix, int nthreads, double* out) {
  if (!out || n_pix < 0 || n_chirps < 0 || n_rx < 1 || nk < 0) return -1;
  if (n_chirps > 0 && (!prof || !tx)) return -1;
  if (n_pix > 0 && !pix) return -1;
  if (!rx && n_rx != 1) return -1;
  if (chirp_s <= 0 || fs_hz <= 0 || nfft < 1) return -1;
  int nt = oracle_threads(nthreads);
  if (nt > n_pix) nt = n_pix > 0 ? n_pix : 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nt);
  bp_job_t* jobs = (bp_job_t*)malloc(sizeof(bp_job_t) * (size_t)nt);
  if (!th || !jobs) { free(th); free(jobs); return -2; }
  for (int i = 0; i < nt; ++i) {
    bp_job_t jb = {prof, n_chirps, n_rx, k0, nk, f0_hz, bandwidth_hz / chirp_s, fs_hz,
                   (double)nfft, tx, rx, doppler, pix, out,
                   (int)((long)n_pix * i / nt), (int)((long)n_pix * (i + 1) / nt), 0};
    jobs[i] = jb;
    pthread_create(&th[i], NULL, bp_worker, &jobs[i]);
  }
  int status = 0;
  for (int i = 0; i < nt; ++i) {
    pthread_join(th[i], NULL);
    if (jobs[i].status) status = jobs[i].status;
  }
  free(th); free(jobs);
  return status;
}

/* ------------------------------------------------------------------------- */
/* Measure D: per-pixel Doppler index shift f_doppler(p) of Alg. 2 */
/* L8, "calculated in advance based on the average vehicle velocity":  */
/*   v_r(p) = legs * <p - q_ref, v_avg> / |p - q_ref|   (Alg. 1 L5, L8, L9 with   */
/*            one velocity for the whole aperture; legs = 2 for TX + RX)        */
/*   f_doppler(p) = (f0 * v_r(p) / c) / (fs / N)         (Alg. 1 L11, in bins)  */
/* A pixel at q_ref gets 0.                                                    */
/* ------------------------------------------------------------------------- */
int oracle_doppler_table(double f0_hz, double fs_hz, int nfft, const double* pix, int n_pix,
                         const double* q_ref, const double* v_avg, double legs, double* out) {
  if (!pix || !q_ref || !v_avg || !out || n_pix < 0 || fs_hz <= 0 || nfft < 1) return -1;
  for (int p = 0; p < n_pix; ++p) {
    const double dx = pix[3 * p] - q_ref[0], dy = pix[3 * p + 1] - q_ref[1], dz = pix[3 * p + 2] - q_ref[2];
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    const double vr = r > 0.0 ? legs * (dx * v_avg[0] + dy * v_avg[1] + dz * v_avg[2]) / r : 0.0;
    out[p] = (f0_hz * vr / ORACLE_C_LIGHT) / (fs_hz / (double)nfft);
  }
  return 0;
}

/* Measure E image -> Cartesian grid "for comparability" (reading
 * A18): for Cartesian pixel (x0 + ix dx, y0 + iy dy) take its polar coordinates about
 * (xc, yc), r = |(x - xc, y - yc)|, th = atan2(x - xc, y - yc) (bearing from +y toward
 * +x), and interpolate the polar image bilinearly in the fractional indices
 * ((th - th0) / dth, (r - r0) / dr), the bearing difference taken modulo 2 pi about the
 * sector centre; pixels outside [0, n_th - 1] x [0, n_r - 1] (up to 1e-9 of an index) are 0.
 *   in  [n_r][n_th][2] (re, im);  out [ny][nx][2]. */
int oracle_polar_to_cartesian(double xc, double yc, double r0, double dr, double th0, double dth,
                              int n_th, int n_r, const double* in, double x0, double y0, double dx,
                              double dy, int nx, int ny, double* out) {
  if (!in || !out || n_th < 1 || n_r < 1 || nx < 0 || ny < 0 || !(dr > 0) || !(dth > 0)) return -1;
  for (int iy = 0; iy < ny; ++iy) {
    for (int ix = 0; ix < nx; ++ix) {
      const double px = x0 + ix * dx - xc, py = y0 + iy * dy - yc;
      /* bearing relative to the sector centre, wrapped into [-pi, pi): bearings are angles
       * (A19), so a sector may cross +-pi and th0 may be given in any period */
      const double half = 0.5 * (n_th - 1) * dth;
      double dbear = atan2(px, py) - (th0 + half);
      dbear -= 2.0 * ORACLE_PI * floor((dbear + ORACLE_PI) / (2.0 * ORACLE_PI));
      double fi = (dbear + half) / dth;
      double fj = (sqrt(px * px + py * py) - r0) / dr;
      double re = 0.0, im = 0.0;
      /* nodes on the sector boundary are inside (1e-9 of an index of rounding slack) */
      if (fi >= -1e-9 && fj >= -1e-9 && fi <= n_th - 1 + 1e-9 && fj <= n_r - 1 + 1e-9) {
        fi = fi < 0.0 ? 0.0 : (fi > n_th - 1 ? n_th - 1 : fi);
        fj = fj < 0.0 ? 0.0 : (fj > n_r - 1 ? n_r - 1 : fj);
        int i0 = (int)floor(fi), j0 = (int)floor(fj);
        if (i0 > n_th - 1) i0 = n_th - 1;
        if (j0 > n_r - 1) j0 = n_r - 1;
        const int i1 = i0 + 1 < n_th ? i0 + 1 : n_th - 1, j1 = j0 + 1 < n_r ? j0 + 1 : n_r - 1;
        const double wi = fi - i0, wj = fj - j0;
        const int idx[4][2] = {{j0, i0}, {j0, i1}, {j1, i0}, {j1, i1}};
        const double w[4] = {(1 - wi) * (1 - wj), wi * (1 - wj), (1 - wi) * wj, wi * wj};
        for (int c = 0; c < 4; ++c) {
          const double* v = in + 2 * ((size_t)idx[c][0] * n_th + idx[c][1]);
          re += w[c] * v[0];
          im += w[c] * v[1];
        }
      }
      out[2 * ((size_t)iy * nx + ix)] = re;
      out[2 * ((size_t)iy * nx + ix) + 1] = im;
    }
  }
  return 0;
}
