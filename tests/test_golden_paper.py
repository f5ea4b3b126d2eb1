"""Pins from numbers the paper prints (tests/golden/paper_numbers.txt, each line cited)."""
import os

import numpy as np

import sarsim

HERE = os.path.dirname(os.path.abspath(__file__))


def _golden():
    out = {}
    with open(os.path.join(HERE, "golden", "paper_numbers.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, val, tol, *cite = line.split()
            out[key] = (float(val), float(tol), " ".join(cite))
    return out


G = _golden()


def _close(key, value):
    v, tol, cite = G[key]
    assert abs(value - v) <= tol, f"{key}: {value} vs paper {v} ({cite})"


def test_paper_grid_convention():
    scn = sarsim.make_config("C0", n_chirps=4)
    g = scn.grid
    _close("pixels_per_axis_30m_2p5cm", g.nx)
    _close("pixels_30m_2p5cm", g.nx * g.ny)
    px = g.pixels()
    _close("plot_xmin_m", px[:, 0].min() - g.dx / 2)
    _close("plot_ymax_m", px[:, 1].max() + g.dy / 2)
    # x from -15 to 15 inclusive (30 m), y from 1 to 31
    assert abs(px[:, 0].max() - 15.0) < 1e-9 and abs(px[:, 1].min() - 1.0) < 1e-12


def test_window_sizes_and_budget():
    _close("window_matrix_bytes", 1201 * 1201 * 1024 * 4)
    _close("window_vector_bytes", 1024 * 4)
    r = sarsim.Radar()
    _close("measurement_time_s", 1024 * r.pri_s)


def test_table1_parameters():
    r = sarsim.Radar()
    _close("f0_hz", r.f0_hz)
    _close("bandwidth_hz", r.bandwidth_hz)
    _close("chirp_s", r.chirp_s)
    _close("pri_s", r.pri_s)
    _close("chirp_rate_hz_per_s", r.bandwidth_hz / r.chirp_s)


def test_config_recipes():
    """Recipes of SURVEY 8(d): C3 arc length and end drop, C2 step, C4 RX offsets."""
    c3 = sarsim.make_config("C3")
    steps = np.linalg.norm(np.diff(c3.tx, axis=0), axis=1)
    assert abs(steps.sum() - 6.556) < 0.01 and steps.min() > 0.63e-3 and steps.max() < 0.97e-3
    assert steps.max() <= sarsim.Radar().wavelength_m / 4          # lambda/4 sampling
    assert -0.28 < c3.tx[:, 1].min() < -0.26
    c2 = sarsim.make_config("C2")
    assert abs(np.diff(c2.tx[:, 0]).mean() - 8 * 106.7e-6) < 1e-12
    c4 = sarsim.make_config("C4", n_chirps=16)
    d = c4.rx[:, :, 0] - c4.tx[:, None, 0]
    assert np.allclose(d[0], 0.005 + np.arange(4) * c4.radar.wavelength_m / 2)
    for name in ("C2", "C3"):
        scn = sarsim.make_config(name, n_chirps=4)
        # isolated targets are >= 1 m from every other scatterer and on pixel centres
        for (j, i) in scn.isolated:
            p = scn.grid.pixel_list(np.array([[j, i]]))[0]
            dist = np.linalg.norm(scn.targets[:, :2] - p[:2], axis=1)
            assert np.sum(dist < 1e-9) == 1 and np.sort(dist)[1] >= 1.0 - 1e-9
