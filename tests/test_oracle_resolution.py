"""Oracle pins from imaging physics (-m "not gpu"): point-spread-function widths against the
textbook resolution formulas and the RX-halving amplitude law of Measure F (
SPEC acceptance 5 and 6).  These fix the oracle's range compression (window, zero padding,
bin spacing), its geometry and its coherent sum over chirps and RX independently of any
retyped formula."""
import math

import numpy as np

import oracle
import sarsim
from sarsim import C_LIGHT, Grid, Radar, Scenario


def _scn(radar, tx, rx, tgt, grid):
    M = tx.shape[0]
    return Scenario("psf", radar, grid, tx, rx, np.asarray([tgt], float), np.asarray([1.0 + 0j]),
                    np.zeros((0, 2), int), np.ones(M, np.float32), 0.0, 0)


def _width_3db(x, a):
    """-3 dB width of the main lobe of |a| sampled at x (linear interpolation of the crossings)."""
    a = np.abs(a) / np.abs(a).max()
    k = int(np.argmax(a))
    lvl = 1 / math.sqrt(2)
    i = k
    while a[i] > lvl:
        i -= 1
    left = x[i] + (lvl - a[i]) / (a[i + 1] - a[i]) * (x[i + 1] - x[i])
    j = k
    while a[j] > lvl:
        j += 1
    right = x[j - 1] + (lvl - a[j - 1]) / (a[j] - a[j - 1]) * (x[j] - x[j - 1])
    return right - left


def test_psf_widths_match_resolution_formulas():
    """Broadside point target at R = 5 m, straight aperture L = 0.5 m (lambda/4 steps):
    range -3 dB width = 1.44 c/(2B) (Hann main lobe, 1.44 bins of the unpadded DFT) and
    azimuth -3 dB width = 0.886 lambda R / (2L) (uniform aperture), each within 3 %."""
    r = Radar()
    lam = r.wavelength_m
    M = int(round(0.5 / (lam / 4))) + 1
    tx = sarsim.straight_track(M, lam / 4)
    L = tx[-1, 0] - tx[0, 0]
    R = 5.0
    # range cut through the target, 5 mm samples
    ys = R + np.arange(-0.4, 0.4001, 0.005)
    grid_r = Grid(0.0, ys[0], 0.0, 1.0, 0.005, 1, len(ys))
    scn = _scn(r, tx, None, (0.0, R, 0.0), grid_r)
    raw = sarsim.simulate_raw(scn).numpy()
    prof = oracle.range_compress(raw, r.fft_len, r.range_window, scn.wsar)
    pr = oracle.backproject(prof, 0, r, tx, None, grid_r.pixels())
    wr = _width_3db(ys, pr)
    wr_theory = 1.44 * C_LIGHT / (2 * r.bandwidth_hz)
    assert abs(wr / wr_theory - 1) < 0.03, (wr, wr_theory)      # measured -0.8 %
    # azimuth cut at the target range, 0.5 mm samples
    xs = np.arange(-0.05, 0.05001, 0.0005)
    grid_a = Grid(xs[0], R, 0.0, 0.0005, 1.0, len(xs), 1)
    pa = oracle.backproject(prof, 0, r, tx, None, grid_a.pixels())
    wa = _width_3db(xs, pa)
    wa_theory = 0.886 * lam * R / (2 * L)
    assert abs(wa / wa_theory - 1) < 0.03, (wa, wa_theory)      # measured -0.2 %


def test_rx_halving_drops_the_peak_by_6_db():
    """Ideal calibrated MIMO array (Measure F): with 8 RX at lambda/2 the coherent
    point-target peak is twice that of the first 4 RX: 20 log10 2 = 6.02 dB (+-0.1 dB)."""
    r = Radar(n_samples=256, fft_len=2048)
    tx = sarsim.straight_track(64, r.wavelength_m / 4)
    rx = sarsim.rx_array(tx, 8, 0.005, r.wavelength_m / 2)
    tgt = (0.02, 4.0, 0.0)
    grid = Grid(0.02, 4.0, 0.0, 1.0, 1.0, 1, 1)
    scn8 = _scn(r, tx, rx, tgt, grid)
    raw8 = sarsim.simulate_raw(scn8).numpy()
    prof8 = oracle.range_compress(raw8, r.fft_len, r.range_window, scn8.wsar)
    p8 = oracle.backproject(prof8, 0, r, tx, rx, grid.pixels())[0]
    p4 = oracle.backproject(np.ascontiguousarray(prof8[:, :4]), 0, r, tx, np.ascontiguousarray(rx[:, :4]),
                            grid.pixels())[0]
    db = 20 * math.log10(abs(p8) / abs(p4))
    assert abs(db - 6.02) < 0.1, db
    # and the peak phase is the target's (A2) for both subsets
    assert abs(np.angle(p8)) < 1e-3 and abs(np.angle(p4)) < 1e-3
