"""Pins for the CPU oracle (-m "not gpu"): each check is fixed by the paper, a closed
form, a special case that reduces to a library routine, or an invariant -- never by
re-calling the oracle's own formula.  See DESIGN.md "Oracle pins" (T1-T9)."""
import math

import numpy as np
import pytest

import oracle
import sarsim
from sarsim import C_LIGHT, Grid, Radar, Scenario


def _tiny_radar(ns=64, z=8, window=1):
    return Radar(n_samples=ns, fft_len=z * ns, range_window=window)


# --------------------------------------------------------------------- T0: primitives
def test_window_matches_numpy_hanning():
    for ns in (2, 3, 16, 255, 512):
        np.testing.assert_allclose(oracle.window(ns, 1), np.hanning(ns), rtol=0, atol=1e-15)
    assert np.all(oracle.window(7, 0) == 1.0)


def test_fft_matches_numpy_and_parseval():
    rng = np.random.default_rng(0)
    for n in (1, 2, 8, 64, 1024, 4096):
        z = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        Z = oracle.fft(z)
        np.testing.assert_allclose(Z, np.fft.fft(z), rtol=0, atol=1e-11 * max(1, np.abs(Z).max()))
        assert abs(np.sum(np.abs(Z) ** 2) / n - np.sum(np.abs(z) ** 2)) < 1e-9 * np.sum(np.abs(z) ** 2)


# --------------------------------------------------------------------- T1: brute-force DFT
@pytest.mark.parametrize("ns", [8, 16, 64])
@pytest.mark.parametrize("z", [1, 4, 8])
@pytest.mark.parametrize("window", [0, 1])
def test_T1_range_compress_fft_equals_literal_dft_and_numpy(ns, z, window):
    rng = np.random.default_rng(ns * 31 + z)
    M, nrx = 3, 2
    raw = rng.standard_normal((M, nrx, ns)).astype(np.float32)
    wsar = rng.uniform(0.2, 1.0, M)
    N = ns * z
    fast = oracle.range_compress(raw, N, window, wsar)
    lit = oracle.range_compress(raw, N, window, wsar, use_dft=True)
    np.testing.assert_allclose(fast, lit, rtol=0, atol=1e-12 * np.abs(lit).max())
    # independent: numpy rfft of the zero-padded windowed row * centring ramp * 2 w_sar/sum(w)
    w = np.hanning(ns) if window == 1 else np.ones(ns)
    if ns == 1:
        w = np.ones(1)
    k = np.arange(N // 2 + 1)
    ramp = np.exp(2j * np.pi * k * (ns - 1) / 2.0 / N)
    ref = np.fft.rfft(raw.astype(np.float64) * w, n=N, axis=-1) * ramp
    ref *= (2.0 * wsar / w.sum())[:, None, None]
    np.testing.assert_allclose(fast, ref, rtol=0, atol=1e-12 * np.abs(ref).max())


def test_T1_crop_and_zero_extension():
    rng = np.random.default_rng(5)
    raw = rng.standard_normal((2, 1, 32)).astype(np.float32)
    N = 128
    full = oracle.range_compress(raw, N, 1)
    crop = oracle.range_compress(raw, N, 1, k0=-3, nk=N // 2 + 10)
    np.testing.assert_array_equal(crop[..., :3], 0)
    np.testing.assert_allclose(crop[..., 3:3 + N // 2 + 1], full, rtol=0, atol=0)
    np.testing.assert_array_equal(crop[..., 3 + N // 2 + 1:], 0)


# --------------------------------------------------------------------- T2: exact-bin tone
@pytest.mark.parametrize("k0,z", [(5, 1), (5, 8), (17, 4), (1, 8)])
def test_T2_exact_bin_tone(k0, z):
    ns, a, phi = 64, 0.7, 1.1
    t = np.arange(ns) - (ns - 1) / 2.0
    x = (a * np.cos(2 * np.pi * k0 * t / ns + phi)).astype(np.float32)
    X = oracle.range_compress(x[None, None, :], ns * z, 0)[0, 0]
    # the closed form only holds for the float32-rounded input to ~1e-7
    assert abs(X[k0 * z] - a * np.exp(1j * phi)) < 2e-7
    for kk in range(0, ns // 2 + 1):
        if kk != k0:
            assert abs(X[kk * z]) < 2e-7


# --------------------------------------------------------------------- helpers
def _scenario(radar, tx, targets, amps, grid, rx=None, wsar=None):
    M = tx.shape[0]
    return Scenario("t", radar, grid, tx, rx, np.asarray(targets, float), np.asarray(amps, complex),
                    np.zeros((0, 2), int), np.ones(M, np.float32) if wsar is None else wsar, 0.0, 0)


def _image(scn, raw=None, pixels=None, doppler=None):
    r = scn.radar
    if raw is None:
        raw = sarsim.simulate_raw(scn).numpy()
    prof = oracle.range_compress(raw, r.fft_len, r.range_window, scn.wsar)
    pix = scn.grid.pixels() if pixels is None else pixels
    return oracle.backproject(prof, 0, r, scn.tx, scn.rx, pix, doppler)


def _interp_gain(radar, kappa):
    """Closed-form linear-interpolation gain of a unit tone: H(d) = sum_t w cos(2 pi d (t-t_c)/N)/sum w
    (real because w is symmetric about t_c, A4), G = (1-f) H(-f) + f H(1-f)."""
    ns, N = radar.n_samples, radar.fft_len
    w = np.hanning(ns) if radar.range_window == 1 else np.ones(ns)
    t = np.arange(ns) - (ns - 1) / 2.0

    def H(d):
        return np.sum(w * np.cos(2 * np.pi * d * t / N)) / w.sum()

    f = kappa - np.floor(kappa)
    return (1 - f) * H(-f) + f * H(1 - f)


# --------------------------------------------------------------------- T3: point target
def test_T3_point_target_C1():
    scn = sarsim.make_config("C1")
    img = _image(scn).reshape(64, 64)
    j, i = np.unravel_index(np.argmax(np.abs(img)), img.shape)
    assert (j, i) == (32, 32)
    p = img[32, 32]
    # sign convention (A2): arg P(p*) = arg a (a wrong sign gives about -1.48 rad here)
    assert abs(np.angle(p * np.conj(scn.amps[0]))) < 1e-6
    r = scn.radar
    a1 = (r.bandwidth_hz / r.chirp_s) * r.fft_len / (C_LIGHT * r.sample_rate_hz)
    d = 2 * np.linalg.norm(scn.tx - scn.targets[0], axis=1)
    G = sum(_interp_gain(r, a1 * dm) for dm in d)
    assert abs(abs(p) - abs(scn.amps[0]) * G) < 1e-6 * G
    assert 0.9975 * 64 < abs(p) <= 64.0 + 1e-9


def test_T3_bistatic_point_target():
    """MIMO form of T3 (TX at the pose, 4 RX ahead of it): the image peaks on the target pixel,
    arg P(p*) = arg a, and |P(p*)| = |a| sum_m sum_n G(a1 (d_tx + d_rx)) with the closed-form
    interpolation gain.  A bistatic path counted as 2 d_tx or 2 d_rx (the monostatic shortcut)
    leaves a phase error of 2 pi f0 (d_rx - d_tx)/c per RX -- radians at these offsets."""
    scn = sarsim.make_config("C1")
    r = scn.radar
    scn.rx = sarsim.rx_array(scn.tx, 4, 0.005, r.wavelength_m / 2.0)
    scn.amps = np.array([0.7 * np.exp(1.1j)])
    img = _image(scn).reshape(64, 64)
    assert np.unravel_index(np.argmax(np.abs(img)), img.shape) == (32, 32)
    p = img[32, 32]
    assert abs(np.angle(p * np.conj(scn.amps[0]))) < 1e-6
    a1 = (r.bandwidth_hz / r.chirp_s) * r.fft_len / (C_LIGHT * r.sample_rate_hz)
    d = np.linalg.norm(scn.tx - scn.targets[0], axis=1)[:, None] + np.linalg.norm(scn.rx - scn.targets[0], axis=2)
    G = sum(_interp_gain(r, a1 * dm) for dm in d.ravel())
    assert abs(abs(p) - abs(scn.amps[0]) * G) < 1e-6 * G
    assert 0.9975 * 0.7 * 64 * 4 < abs(p) <= 0.7 * 64 * 4 + 1e-9


def test_T3_argmax_random_single_targets():
    """Matched-filter argmax lands on the scatterer's pixel (SPEC-style property, 12 seeds)."""
    for seed in range(12):
        scn = sarsim.small_config(n_chirps=32, ns=64, nx=24, ny=16, seed=100 + seed,
                                  curved=bool(seed % 2))
        scn.targets = scn.targets[:1]
        scn.amps = scn.amps[:1]
        img = np.abs(_image(scn)).reshape(scn.grid.ny, scn.grid.nx)
        assert tuple(np.unravel_index(np.argmax(img), img.shape)) == tuple(scn.isolated[0])


# --------------------------------------------------------------------- T4: flat profile
@pytest.mark.parametrize("bistatic", [False, True])
def test_T4_flat_profile_gives_exact_coherent_sum(bistatic):
    r = _tiny_radar(ns=256)   # Nyquist range 20.6 m covers the 6.1 m pixel
    M, nrx = 40, (3 if bistatic else 1)
    tx = sarsim.curved_track(M, r.pri_s, 6, 9, 7.0)
    rx = sarsim.rx_array(tx, nrx, 0.005, 0.002) if bistatic else None
    p = np.array([0.37, 6.1, 0.0])
    a = 0.8 * np.exp(0.3j)
    dtx = np.linalg.norm(tx - p, axis=1)
    drx = np.linalg.norm(rx - p, axis=2) if bistatic else dtx[:, None]
    d = dtx[:, None] + drx
    nk = r.fft_len // 2 + 1
    prof = np.repeat((a * np.exp(-2j * np.pi * r.f0_hz * d / C_LIGHT))[:, :, None], nk, axis=2)
    P = oracle.backproject(prof, 0, r, tx, rx, p[None, :])[0]
    assert abs(P - a * M * nrx) < 1e-10 * M * nrx


# --------------------------------------------------------------------- T5: exact bin
def test_T5_circular_track_exact_bin_gives_N_a():
    r = _tiny_radar(ns=64, z=8, window=0)
    a1 = r.bandwidth_hz * (r.fft_len // r.n_samples) / C_LIGHT
    kappa = 8 * 20                      # a native bin: no leakage with a rectangular window
    R = kappa / (2 * a1)
    M = 50
    ang = np.linspace(-0.4, 0.4, M) - np.pi / 2
    tgt = np.array([0.1, 5.0, 0.0])
    tx = np.stack([tgt[0] + R * np.cos(ang), tgt[1] + R * np.sin(ang), np.zeros(M)], 1)
    grid = Grid(0.1 - 0.04, 5.0 - 0.04, 0.0, 0.02, 0.02, 5, 5)
    a = 0.6 * np.exp(-2.0j)
    scn = _scenario(r, tx, [tgt], [a], grid)
    img = _image(scn).reshape(5, 5)
    assert abs(img[2, 2] - a * M) < 1e-6 * M   # float32 raw rounding bounds it to ~1e-7
    assert np.argmax(np.abs(img)) == 12


# --------------------------------------------------------------------- T6: permutation
def test_T6_chirp_permutation_invariance():
    scn = sarsim.small_config(n_chirps=40, ns=64, nx=16, ny=12, curved=True, n_rx=2, seed=4)
    scn.wsar = np.linspace(0.3, 1.0, 40).astype(np.float32)
    raw = sarsim.simulate_raw(scn).numpy()
    img = _image(scn, raw)
    perm = np.random.default_rng(1).permutation(40)
    scn2 = _scenario(scn.radar, scn.tx[perm], scn.targets, scn.amps, scn.grid, scn.rx[perm], scn.wsar[perm])
    img2 = _image(scn2, raw[perm])
    assert np.abs(img2 - img).max() < 1e-12 * np.abs(img).max()


# --------------------------------------------------------------------- T7: translation
def test_T7_translation_invariance():
    scn = sarsim.small_config(n_chirps=32, ns=64, nx=12, ny=10, seed=7)
    raw = sarsim.simulate_raw(scn).numpy()
    img = _image(scn, raw)
    sh = np.array([1000.0, 1000.0, 0.0])
    g = scn.grid
    grid2 = Grid(g.x0 + 1000.0, g.y0 + 1000.0, 0.0, g.dx, g.dy, g.nx, g.ny)
    scn2 = _scenario(scn.radar, scn.tx + sh, scn.targets + sh, scn.amps, grid2)
    img2 = _image(scn2, raw)
    assert np.abs(img2 - img).max() < 1e-8 * np.abs(img).max()


# --------------------------------------------------------------------- T8: linearity
def test_T8_linearity_and_scaling():
    scn = sarsim.small_config(n_chirps=24, ns=64, nx=12, ny=10, seed=9)
    ra = sarsim.simulate_raw(scn, targets=scn.targets[:1], amps=scn.amps[:1]).numpy().astype(np.float64)
    rb = sarsim.simulate_raw(scn, targets=scn.targets[1:], amps=scn.amps[1:]).numpy().astype(np.float64)
    # float32 is the raw format: use inputs exactly representable so sums stay exact
    ra = np.round(ra * 1024) / 1024
    rb = np.round(rb * 1024) / 1024
    ia = _image(scn, ra.astype(np.float32))
    ib = _image(scn, rb.astype(np.float32))
    iab = _image(scn, (ra + rb).astype(np.float32))
    assert np.abs(iab - ia - ib).max() < 1e-12 * np.abs(iab).max()
    i2 = _image(scn, (2.0 * ra).astype(np.float32))
    assert np.abs(i2 - 2 * ia).max() < 1e-12 * np.abs(i2).max()


# --------------------------------------------------------------------- T9: degenerate
def test_T9_zero_input_and_pixel_on_antenna():
    scn = sarsim.small_config(n_chirps=8, ns=32, nx=6, ny=5, seed=1)
    raw = np.zeros((8, 1, 32), np.float32)
    assert np.all(_image(scn, raw) == 0)
    raw = sarsim.simulate_raw(scn).numpy()
    v = _image(scn, raw, pixels=scn.tx[3][None, :])
    assert np.all(np.isfinite(v))
    # no chirps -> empty sum
    r = scn.radar
    out = oracle.backproject(np.zeros((0, 1, 5)), 0, r, np.zeros((0, 3)), None, scn.grid.pixels()[:3])
    assert np.all(out == 0)


def test_crop_too_small_is_reported():
    scn = sarsim.small_config(n_chirps=4, ns=128, nx=4, ny=4, seed=1)
    r = scn.radar
    prof = oracle.range_compress(sarsim.simulate_raw(scn).numpy(), r.fft_len, 1, k0=0, nk=10)
    with pytest.raises(RuntimeError, match="crop"):
        oracle.backproject(prof, 0, r, scn.tx, None, scn.grid.pixels())


def test_thread_count_determinism():
    scn = sarsim.small_config(n_chirps=16, ns=64, nx=10, ny=7, seed=2)
    r = scn.radar
    prof = oracle.range_compress(sarsim.simulate_raw(scn).numpy(), r.fft_len, 1)
    a = oracle.backproject(prof, 0, r, scn.tx, None, scn.grid.pixels(), nthreads=1)
    b = oracle.backproject(prof, 0, r, scn.tx, None, scn.grid.pixels(), nthreads=5)
    np.testing.assert_array_equal(a, b)


# --------------------------------------------------------------------- Measure D (NEXT-3)
def test_doppler_table_closed_forms():
    """SPEC-style examples: v = 0 -> 0; broadside -> 0; v = (10, 0) m/s and a
    pixel along +x -> v_r = 20 m/s -> f0 20 / c Hz = (that) / (fs / N) bins."""
    r = Radar()
    pix = np.array([[25.0, 0.0, 0.0], [0.0, 7.0, 0.0], [-3.0, 0.0, 0.0], [0.0, 0.0, 0.0]])
    assert np.all(oracle.doppler_table(r, pix, [0, 0, 0], [0, 0, 0]) == 0)
    d = oracle.doppler_table(r, pix, [0, 0, 0], [10.0, 0, 0])
    fd_bins = (r.f0_hz * 20.0 / C_LIGHT) / (r.sample_rate_hz / r.fft_len)
    assert abs(d[0] - fd_bins) < 1e-12 * fd_bins and abs(fd_bins - 4.18628) < 1e-4
    assert d[1] == 0 and abs(d[2] + fd_bins) < 1e-12 * fd_bins and d[3] == 0


def test_doppler_term_corrects_the_range_shift():
    """Doppler materiality: a squinted target seen from a moving
    platform appears shifted in range by f_D/mu c/2 without the f_doppler(p) term; with the
    Measure D table (aperture-centre position, average velocity) the peak is back on the
    target pixel and the coherent gain is restored."""
    r = Radar(n_samples=256, fft_len=2048)
    M = 160
    tx = sarsim.straight_track(M, 9.0 * r.pri_s)
    tgt = np.array([2.5, 2.5, 0.0])                        # 45 degrees squint, v_r ~ 12.7 m/s
    grid = Grid(2.5 - 0.3, 2.5 - 0.3, 0.0, 0.01, 0.01, 61, 61)
    scn = _scenario(r, tx, [tgt], [1.0 + 0j], grid)
    raw = sarsim.simulate_raw(scn, doppler=True).numpy()
    prof = oracle.range_compress(raw, r.fft_len, 1, scn.wsar)
    pix = grid.pixels()
    q_ref = tx.mean(0)
    v_avg = sarsim.track_velocity(scn).mean(0)
    dop = oracle.doppler_table(r, pix, q_ref, v_avg)
    plain = np.abs(oracle.backproject(prof, 0, r, tx, None, pix)).reshape(61, 61)
    fixed = np.abs(oracle.backproject(prof, 0, r, tx, None, pix, doppler=dop)).reshape(61, 61)
    jt = it = 30
    jp, ip = np.unravel_index(np.argmax(plain), plain.shape)
    jf, i_f = np.unravel_index(np.argmax(fixed), fixed.shape)
    # expected one-way range shift f_D / mu * c / 2 = dop / a1 / 2
    a1 = r.bandwidth_hz * (r.fft_len // r.n_samples) / C_LIGHT
    shift = dop[jt * 61 + it] / a1 / 2
    assert 0.03 < shift < 0.06
    moved = np.hypot(*(pix[jp * 61 + ip, :2] - q_ref[:2])) - np.hypot(*(tgt[:2] - q_ref[:2]))
    assert abs(moved - shift) < 0.015          # closing target: higher beat -> appears farther
    assert (jf, i_f) == (jt, it)
    assert fixed[jt, it] > 0.99 * 0.9975 * M and fixed.max() > plain.max()
