"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no range compression, no
back-projection).  It only builds, from a seed:
  * radar parameters (Table 1, plus readings A4-A7 in DESIGN.md),
  * per-chirp antenna phase centres along straight or curved tracks (the
    "non-equidistant ... curved track" of the north star; stop-and-go, A10),
  * point-scatterer scenes modelled on the Fig. 1 regions (pole, wall, yard,
    P:L112-114) plus isolated, pixel-centred calibration points,
  * the real FMCW beat samples those scenes produce (the forward model the
    paper's signal s comes from; see ``simulate_raw``),
  * optional AWGN drawn from a seeded generator,
  * the pixel grid (pixel (i, j) at (x0 + i dx, y0 + j dy, z0)).

Recipes for configs C0-C5 follow SURVEY.md section 8(d) and are restated in
DESIGN.md ("Input recipe").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

C_LIGHT = 299792458.0


@dataclass(frozen=True)
class Radar:
    """Table 1 + the two quantities the paper omits (A5)."""
    f0_hz: float = 76.6e9            # centre frequency of the sampled sweep (A4)
    bandwidth_hz: float = 931e6      # B
    chirp_s: float = 102.4e-6        # T_P
    pri_s: float = 106.7e-6          # T_P0
    n_samples: int = 512             # Ns (A5)
    fft_len: int = 4096              # N_fft = Z * Ns, Z = 8 (A6)
    range_window: int = 1            # 0 rectangular, 1 symmetric Hann (A6)

    @property
    def sample_rate_hz(self) -> float:
        return self.n_samples / self.chirp_s

    @property
    def wavelength_m(self) -> float:
        return C_LIGHT / self.f0_hz


@dataclass(frozen=True)
class Grid:
    x0: float
    y0: float
    z0: float
    dx: float
    dy: float
    nx: int
    ny: int

    def pixels(self, rows=None, cols=None) -> np.ndarray:
        """Pixel centres [n][3] (row-major j, i) for the given row/col index arrays."""
        j = np.arange(self.ny) if rows is None else np.asarray(rows)
        i = np.arange(self.nx) if cols is None else np.asarray(cols)
        jj, ii = np.meshgrid(j, i, indexing="ij")
        out = np.empty(jj.shape + (3,), np.float64)
        out[..., 0] = self.x0 + ii * self.dx
        out[..., 1] = self.y0 + jj * self.dy
        out[..., 2] = self.z0
        return out.reshape(-1, 3)

    def pixel_list(self, idx_ji: np.ndarray) -> np.ndarray:
        idx = np.asarray(idx_ji).reshape(-1, 2)
        out = np.empty((idx.shape[0], 3), np.float64)
        out[:, 0] = self.x0 + idx[:, 1] * self.dx
        out[:, 1] = self.y0 + idx[:, 0] * self.dy
        out[:, 2] = self.z0
        return out


@dataclass(frozen=True)
class PolarGrid:
    """Measure E polar grid: pixel (i, j) at (xc + r_j sin th_i, yc + r_j cos th_i, zc),
    r_j = r0 + j dr, th_i = th0 + i dth (from +y toward +x); images [n_r][n_th]."""
    xc: float
    yc: float
    zc: float
    r0: float
    dr: float
    th0: float
    dth: float
    n_th: int
    n_r: int

    @property
    def nx(self) -> int:
        return self.n_th

    @property
    def ny(self) -> int:
        return self.n_r

    def pixels(self, rows=None, cols=None) -> np.ndarray:
        j = np.arange(self.n_r) if rows is None else np.asarray(rows)
        i = np.arange(self.n_th) if cols is None else np.asarray(cols)
        jj, ii = np.meshgrid(j, i, indexing="ij")
        r = self.r0 + jj * self.dr
        th = self.th0 + ii * self.dth
        out = np.empty(jj.shape + (3,), np.float64)
        out[..., 0] = self.xc + r * np.sin(th)
        out[..., 1] = self.yc + r * np.cos(th)
        out[..., 2] = self.zc
        return out.reshape(-1, 3)

    def pixel_list(self, idx_ji: np.ndarray) -> np.ndarray:
        idx = np.asarray(idx_ji).reshape(-1, 2)
        r = self.r0 + idx[:, 0] * self.dr
        th = self.th0 + idx[:, 1] * self.dth
        return np.stack([self.xc + r * np.sin(th), self.yc + r * np.cos(th), np.full(len(r), self.zc)], 1)


def polar_recipe(radar: Radar, centre, aperture_m: float, r_min: float, r_max: float,
                 th_min: float, th_max: float, factor: float = 2.5) -> PolarGrid:
    """Polar grid a `factor` finer than the PSF: range spacing
    dr = (c / 2B) / factor; bearing spacing from the azimuth resolution lambda R / (2 L) at
    r_max, r_max dth = lambda r_max / (2 L factor) (uniform dth)."""
    if factor < 2:
        raise ValueError("oversampling factor must be >= 2 (point targets, P:L326)")
    dr = C_LIGHT / (2 * radar.bandwidth_hz) / factor
    dth = radar.wavelength_m / (2 * aperture_m * factor)
    n_r = int(np.floor((r_max - r_min) / dr)) + 1
    n_th = int(np.floor((th_max - th_min) / dth)) + 1
    return PolarGrid(float(centre[0]), float(centre[1]), float(centre[2]), r_min, dr, th_min, dth, n_th, n_r)


@dataclass
class Scenario:
    name: str
    radar: Radar
    grid: Grid
    tx: np.ndarray                    # [M][3] float64
    rx: np.ndarray | None             # [M][N_rx][3] float64, None = monostatic
    targets: np.ndarray               # [K][3] float64
    amps: np.ndarray                  # [K] complex128
    isolated: np.ndarray              # [I][2] (j, i) pixel indices of isolated targets
    wsar: np.ndarray                  # [M] float32
    noise_sigma: float = 0.0
    seed: int = 0
    notes: dict = field(default_factory=dict)

    @property
    def n_chirps(self) -> int:
        return self.tx.shape[0]

    @property
    def n_rx(self) -> int:
        return 1 if self.rx is None else self.rx.shape[1]

    @property
    def updates(self) -> int:
        return self.grid.nx * self.grid.ny * self.n_chirps * self.n_rx

    def antenna_box(self, margin: float = 0.0):
        pts = self.tx if self.rx is None else np.concatenate([self.tx, self.rx.reshape(-1, 3)])
        return pts.min(0) - margin, pts.max(0) + margin


# ----------------------------------------------------------------------------- tracks
def straight_track(n_chirps: int, step_m: float, centre_index: float | None = None,
                   y: float = 0.0) -> np.ndarray:
    """Equidistant straight track along +x at y, z = 0 (radar looks toward +y)."""
    c = (n_chirps - 1) / 2.0 if centre_index is None else centre_index
    q = np.zeros((n_chirps, 3))
    q[:, 0] = (np.arange(n_chirps) - c) * step_m
    q[:, 1] = y
    return q


def curved_track(n_chirps: int, pri_s: float, v0: float, v1: float, radius: float) -> np.ndarray:
    """Arc of ``radius`` bending away from the scene (toward -y), tangent +x at the
    origin, speed ramping linearly v0 -> v1 over the aperture (non-equidistant)."""
    v = v0 + (v1 - v0) * np.arange(n_chirps) / max(n_chirps - 1, 1)
    s = np.concatenate([[0.0], np.cumsum(v[:-1] * pri_s)])
    s -= 0.5 * (s[0] + s[-1])
    q = np.zeros((n_chirps, 3))
    q[:, 0] = radius * np.sin(s / radius)
    q[:, 1] = -radius * (1.0 - np.cos(s / radius))
    return q


def rx_array(tx: np.ndarray, n_rx: int, first_offset: float, spacing: float) -> np.ndarray:
    rx = np.repeat(tx[:, None, :], n_rx, axis=1).copy()
    rx[:, :, 0] += first_offset + spacing * np.arange(n_rx)[None, :]
    return rx


# ----------------------------------------------------------------------------- scenes
def _snap(grid: Grid, x, y):
    i = np.rint((np.asarray(x) - grid.x0) / grid.dx).astype(np.int64)
    j = np.rint((np.asarray(y) - grid.y0) / grid.dy).astype(np.int64)
    return j, i


def fig1_scene(rng: np.random.Generator, grid: Grid, n_isolated: int,
               iso_box, extra_isolated: int = 0, extra_box=None):
    """Pole / wall / yard (P:L112-114 rectangles) + isolated pixel-centred points."""
    pos, amp = [], []
    # pole: strongest scatterer, a = 1 (global argmax by a 10 % margin, A15)
    pos.append((3.25, 7.85)); amp.append(1.0 + 0j)
    # wall: 133 points on y = 11.20, x in [-5.5, 1.1] every 5 cm, |a| = 0.3, random phase
    for x in np.linspace(-5.5, 1.1, 133):
        pos.append((x, 11.20)); amp.append(0.3 * np.exp(1j * rng.uniform(0, 2 * np.pi)))
    # yard: 256 points uniform in [-6.5, -1.2] x [11.2, 12.6], |a| ~ Rayleigh(0.05)
    for _ in range(256):
        pos.append((rng.uniform(-6.5, -1.2), rng.uniform(11.2, 12.6)))
        amp.append(rng.rayleigh(0.05) * np.exp(1j * rng.uniform(0, 2 * np.pi)))
    iso = []

    def place(count, box):
        tries = 0
        while count > 0:
            tries += 1
            if tries > 200000:
                raise RuntimeError("could not place isolated targets")
            x = rng.uniform(box[0], box[1]); y = rng.uniform(box[2], box[3])
            j, i = _snap(grid, x, y)
            x = grid.x0 + i * grid.dx; y = grid.y0 + j * grid.dy
            if min(math.hypot(x - px, y - py) for px, py in pos) < 1.0:
                continue
            pos.append((x, y))
            amp.append(rng.uniform(0.5, 0.9) * np.exp(1j * rng.uniform(0, 2 * np.pi)))
            iso.append((j, i))
            count -= 1

    # the pole is isolated too (nothing within 1 m)
    iso.append(tuple(int(v) for v in _snap(grid, 3.25, 7.85)))
    place(n_isolated, iso_box)
    if extra_isolated:
        place(extra_isolated, extra_box)
    p = np.zeros((len(pos), 3)); p[:, :2] = np.asarray(pos)
    return p, np.asarray(amp, np.complex128), np.asarray(iso, np.int64)


# ----------------------------------------------------------------------------- configs
def make_config(name: str, n_chirps: int | None = None, seed: int | None = None,
                wsar: str = "rect", noise_sigma: float | None = None) -> Scenario:
    """Configs of BASELINE.json (C1-C5) + C0 (the paper's 1201^2 grid), SURVEY 8(d)."""
    name = name.upper()
    if name == "C1":
        radar = Radar(n_samples=256, fft_len=2048)
        M = n_chirps or 64
        lam = radar.wavelength_m
        tx = straight_track(M, lam / 4.0, centre_index=M // 2)
        grid = Grid(-0.64, 4.36, 0.0, 0.02, 0.02, 64, 64)
        tgt = np.array([[0.0, 5.00, 0.0]]); amp = np.array([1.0 + 0j])
        iso = np.array([[32, 32]])
        scn = Scenario("C1", radar, grid, tx, None, tgt, amp, iso, None, 0.0, seed or 1)
    elif name in ("C6", "C6P"):
        # The paper's own measurement (reading A1): ONE chirp sequence of N_m = 1024 chirps
        # (109.3 ms) x 8 RX (Measure F) = 8192 aperture samples, on the paper's
        # 1201^2 grid at 2.5 cm (C6) or on the Measure E polar grid (C6p).  A slow straight pass
        # (0.75 m/s, aperture 8.2 cm) -- the aperture for which the recipe's grid has the
        # paper's 165,061 pixels (reading A19).
        radar = Radar()
        M = n_chirps or 1024
        tx = straight_track(M, 0.75 * radar.pri_s)
        rx = rx_array(tx, 8, 0.005, radar.wavelength_m / 2.0)
        grid = Grid(-15.0, 1.0, 0.0, 0.025, 0.025, 1201, 1201)
        sd = seed or 7
        rng = np.random.default_rng(sd)
        tgt, amp, iso = fig1_scene(rng, grid, 32, (-14.5, 14.5, 1.5, 12.5), 64, (-14.5, 14.5, 1.5, 30.5))
        scn = Scenario(name if name == "C6" else "C6p", radar, grid, tx, rx, tgt, amp, iso, None, 0.05, sd)
        if name == "C6P":
            th = float(np.arctan2(15.0, 1.0))
            L = float(np.linalg.norm(tx[-1] - tx[0]))
            scn.grid = polar_recipe(radar, tx.mean(0), L, 1.0, float(np.hypot(15.0, 31.0)), -th, th, 2.5)
            scn.isolated = np.zeros((0, 2), np.int64)
    elif name in ("C2", "C0", "C5"):
        radar = Radar()
        # C5: one long straight track of 8192 + 15 hops of 1024 chirps (16 frames)
        M = n_chirps or (8192 + 15 * 1024 if name == "C5" else 8192)
        step = 8.0 * radar.pri_s
        tx = straight_track(M, step)
        if name == "C2":
            grid = Grid(-15.0, 1.0, 0.0, 0.01, 0.01, 3000, 1200)
        elif name == "C0":
            grid = Grid(-15.0, 1.0, 0.0, 0.025, 0.025, 1201, 1201)
        else:
            grid = Grid(-15.0, 1.0, 0.0, 0.01, 0.01, 3000, 1200)
        sd = seed or {"C2": 2, "C0": 6, "C5": 5}[name]
        rng = np.random.default_rng(sd)
        tgt, amp, iso = fig1_scene(rng, grid, 32, (-14.5, 14.5, 1.5, 12.5))
        scn = Scenario(name, radar, grid, tx, None, tgt, amp, iso, None, 0.05, sd)
    elif name == "C3":
        radar = Radar()
        M = n_chirps or 8192
        tx = curved_track(M, radar.pri_s, 6.0, 9.0, 20.0)
        grid = Grid(-15.0, 1.0, 0.0, 0.01, 0.01, 3000, 3000)
        sd = seed or 3
        rng = np.random.default_rng(sd)
        tgt, amp, iso = fig1_scene(rng, grid, 32, (-14.5, 14.5, 1.5, 12.5),
                                   64, (-14.5, 14.5, 1.5, 30.5))
        scn = Scenario("C3", radar, grid, tx, None, tgt, amp, iso, None, 0.05, sd)
    elif name == "C4":
        radar = Radar()
        M = n_chirps or 8192
        tx = straight_track(M, 8.0 * radar.pri_s)
        rx = rx_array(tx, 4, 0.005, radar.wavelength_m / 2.0)
        grid = Grid(-15.0, 1.0, 0.0, 0.005, 0.005, 6000, 6000)
        sd = seed or 4
        rng = np.random.default_rng(sd)
        tgt, amp, iso = fig1_scene(rng, grid, 32, (-14.5, 14.5, 1.5, 12.5),
                                   64, (-14.5, 14.5, 1.5, 30.5))
        scn = Scenario("C4", radar, grid, tx, rx, tgt, amp, iso, None, 0.05, sd)
    else:
        raise ValueError(f"unknown config {name}")
    if noise_sigma is not None:
        scn.noise_sigma = noise_sigma
    M = scn.n_chirps
    if wsar == "rect":
        scn.wsar = np.ones(M, np.float32)
    elif wsar == "hann":
        u = np.arange(M) / max(M - 1, 1)
        scn.wsar = (0.5 - 0.5 * np.cos(2 * np.pi * u)).astype(np.float32)
    else:
        raise ValueError(wsar)
    return scn


def c5_frames(scn: Scenario, hop: int = 1024, aperture: int = 8192, n_frames: int | None = None):
    """C5 streaming frames: frame f uses chirps [f hop, f hop + aperture) and the
    C2 grid (3000 x 1200 at 1 cm) re-centred in x on the frame's aperture centre, snapped to the
    pixel pitch.  One frame per hop = one paper measurement of N_m T_P0 = 109.3 ms.
    Returns [(chirp0, Grid)]."""
    g = scn.grid
    total = (scn.n_chirps - aperture) // hop + 1
    n = total if n_frames is None else min(n_frames, total)
    frames = []
    for f in range(n):
        c0 = f * hop
        xc = float(np.mean(scn.tx[c0:c0 + aperture, 0]))
        x0 = round((xc - 0.5 * (g.nx - 1) * g.dx) / g.dx) * g.dx
        frames.append((c0, Grid(x0, g.y0, g.z0, g.dx, g.dy, g.nx, g.ny)))
    return frames


def small_config(n_chirps=48, ns=128, nx=40, ny=24, n_rx=1, seed=11, curved=False,
                 noise_sigma=0.0, grid_dx=0.02) -> Scenario:
    """A seconds-scale scene for CPU tests: a few isolated targets near 4-6 m range."""
    radar = Radar(n_samples=ns, fft_len=8 * ns)
    rng = np.random.default_rng(seed)
    if curved:
        tx = curved_track(n_chirps, radar.pri_s, 6.0, 9.0, 5.0)
    else:
        tx = straight_track(n_chirps, radar.wavelength_m / 4.0)
    rx = None if n_rx == 1 else rx_array(tx, n_rx, 0.005, radar.wavelength_m / 2.0)
    grid = Grid(-0.4, 4.2, 0.0, grid_dx, grid_dx, nx, ny)
    pts, amps, iso = [], [], []
    for k in range(3):
        mx, my = min(6, nx // 4), min(3, ny // 4)
        i = int(rng.integers(mx, nx - mx)); j = int(rng.integers(my, ny - my))
        pts.append((grid.x0 + i * grid.dx, grid.y0 + j * grid.dy, 0.0))
        amps.append(rng.uniform(0.5, 1.0) * np.exp(1j * rng.uniform(0, 2 * np.pi)))
        iso.append((j, i))
    return Scenario("small", radar, grid, tx, rx, np.asarray(pts), np.asarray(amps, np.complex128),
                    np.asarray(iso), np.ones(n_chirps, np.float32), noise_sigma, seed)


def polar_small_config(n_chirps=64, ns=256, n_th=70, n_r=40, n_rx=1, seed=31, curved=False,
                       r0=4.2, dr=0.02, th0=-0.18, dth=0.005, centre=(0.0, 0.0, 0.0)) -> Scenario:
    """Seconds-scale scene on a polar grid (Measure E) about the aperture
    centre: three isolated point targets on polar nodes."""
    radar = Radar(n_samples=ns, fft_len=8 * ns)
    rng = np.random.default_rng(seed)
    if curved:
        tx = curved_track(n_chirps, radar.pri_s, 6.0, 9.0, 5.0)
    else:
        tx = straight_track(n_chirps, radar.wavelength_m / 4.0)
    rx = None if n_rx == 1 else rx_array(tx, n_rx, 0.005, radar.wavelength_m / 2.0)
    grid = PolarGrid(centre[0], centre[1], centre[2], r0, dr, th0, dth, n_th, n_r)
    iso, amps = [], []
    for k in range(3):
        mi, mj = min(6, n_th // 4), min(3, n_r // 4)
        iso.append((int(rng.integers(mj, n_r - mj)), int(rng.integers(mi, n_th - mi))))
        amps.append(rng.uniform(0.5, 1.0) * np.exp(1j * rng.uniform(0, 2 * np.pi)))
    iso = np.asarray(iso)
    return Scenario("polar_small", radar, grid, tx, rx, grid.pixel_list(iso), np.asarray(amps, np.complex128),
                    iso, np.ones(n_chirps, np.float32), 0.0, seed)


# ----------------------------------------------------------------------------- raw beat
def track_velocity(scn: Scenario) -> np.ndarray:
    """Per-chirp platform velocity [M][3] (central differences of the TX track over T_P0)."""
    q = scn.tx
    if q.shape[0] < 2:
        return np.zeros_like(q)
    v = np.gradient(q, axis=0) / scn.radar.pri_s
    return v


def simulate_raw(scn: Scenario, device: str = "cpu", chirp_block: int = 64,
                 targets=None, amps=None, doppler: bool = False):
    """Real FMCW beat samples float32 [M][N_rx][Ns] of a stop-and-go point scene.

    For scatterer k with complex reflectivity a_k and two-way path
    d = |p_k - q_tx(m)| + |p_k - q_rx(m,n)|, tau = d/c (Alg. 1 L10):
        x[t] = sum_k |a_k| cos(2 pi mu tau (t - t_c)/fs - 2 pi f0 tau + arg a_k)
    with mu = B/T_P, t_c = (Ns-1)/2 and f0 the centre frequency (A4);
    the positive-frequency component carries phase -2 pi f0 tau (A2).  No range
    decay, no residual video phase (A11).  Stop-and-go by default; with ``doppler=True``
    the beat frequency carries the Doppler term of Alg. 1 L5, L8, L9, L11:
    mu tau + f0 (v_tx + v_rx)/c with v_tx = <p - q_tx, v(m)>/|p - q_tx| (same for RX) and
    v(m) the platform velocity (A10).
    AWGN of std ``noise_sigma`` per sample from a seeded torch generator.
    Computed in float64 (torch, on ``device``), returned as a float32 torch tensor.
    """
    import torch

    r = scn.radar
    tg = scn.targets if targets is None else np.asarray(targets)
    am = scn.amps if amps is None else np.asarray(amps)
    M, nrx, ns = scn.n_chirps, scn.n_rx, r.n_samples
    dev = torch.device(device)
    f64 = torch.float64
    P = torch.as_tensor(tg, dtype=f64, device=dev)                      # [K,3]
    mag = torch.as_tensor(np.abs(am), dtype=f64, device=dev)             # [K]
    arg = torch.as_tensor(np.angle(am), dtype=f64, device=dev)           # [K]
    tx = torch.as_tensor(scn.tx, dtype=f64, device=dev)
    rx = None if scn.rx is None else torch.as_tensor(scn.rx, dtype=f64, device=dev)
    mu = r.bandwidth_hz / r.chirp_s
    fs = r.sample_rate_hz
    tcen = torch.arange(ns, dtype=f64, device=dev) - 0.5 * (ns - 1)
    out = torch.empty((M, nrx, ns), dtype=torch.float32, device=dev)
    kb = max(1, min(len(tg), 4_000_000 // max(1, chirp_block * nrx * ns)))
    for m0 in range(0, M, chirp_block):
        m1 = min(M, m0 + chirp_block)
        dtx = torch.linalg.norm(P[None, :, :] - tx[m0:m1, None, :], dim=-1)        # [b,K]
        if rx is None:
            d = (2.0 * dtx)[:, None, :]                                              # [b,1,K]
        else:
            drx = torch.linalg.norm(P[None, None, :, :] - rx[m0:m1, :, None, :], dim=-1)
            d = dtx[:, None, :] + drx                                                # [b,n,K]
        tau = d / C_LIGHT
        cyc_f0 = r.f0_hz * tau
        ph0 = -2.0 * math.pi * (cyc_f0 - torch.floor(cyc_f0)) + arg                 # [b,n,K]
        fb = mu * tau / fs                                                           # cycles/sample
        if doppler:
            vel = torch.as_tensor(track_velocity(scn)[m0:m1], dtype=f64, device=dev)  # [b,3]
            ut = (P[None, :, :] - tx[m0:m1, None, :]) / dtx[..., None]               # [b,K,3]
            v_tx = (ut * vel[:, None, :]).sum(-1)                                     # Alg. 1 L5
            if rx is None:
                v = (2.0 * v_tx)[:, None, :]
            else:
                ur = (P[None, None, :, :] - rx[m0:m1, :, None, :]) / drx[..., None]
                v = v_tx[:, None, :] + (ur * vel[:, None, None, :]).sum(-1)           # Alg. 1 L8, L9
            fb = fb + r.f0_hz * v / C_LIGHT / fs                                      # Alg. 1 L11
        acc = torch.zeros((m1 - m0, nrx, ns), dtype=f64, device=dev)
        for k0 in range(0, len(tg), kb):
            k1 = min(len(tg), k0 + kb)
            ph = 2.0 * math.pi * fb[..., k0:k1, None] * tcen + ph0[..., k0:k1, None]
            acc += (mag[k0:k1, None] * torch.cos(ph)).sum(dim=-2)
        out[m0:m1] = acc.to(torch.float32)
    if scn.noise_sigma > 0:
        g = torch.Generator(device="cpu").manual_seed(int(scn.seed) * 7919 + 17)
        noise = torch.randn((M, nrx, ns), generator=g, dtype=torch.float32) * float(scn.noise_sigma)
        out += noise.to(dev)
    return out
