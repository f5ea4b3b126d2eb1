"""C-ABI boundary on CPU (-m "not gpu"): the library builds and loads, exports every symbol
include/sar_bp.h declares, and its host-side plan maths (no device needed) is right."""
import ctypes
import math
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import sarsim
from paper_2306_09784_b200 import _build, sar

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return sar.load()


def _declared_symbols():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", fn)).read()
            txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
            names |= set(re.findall(r"\b(sar_[a-z_0-9]+)\s*\(", txt))
    return names


def test_exports_every_declared_symbol(lib):
    names = _declared_symbols()
    assert {"sar_plan_create", "sar_range_compress", "sar_backproject", "sar_destroy"} <= names
    for n in names:
        assert hasattr(lib, n), f"libsar.so does not export {n}"
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def _params(scn, **kw):
    r = scn.radar
    rp = sar.radar_params(r, scn.n_chirps, scn.n_rx)
    for k, v in kw.items():
        setattr(rp, k, v)
    lo, hi = scn.antenna_box()
    return rp, sar.grid_params(scn.grid), sar.box_params(lo, hi)


def test_plan_geometry_constants_and_crop(lib):
    scn = sarsim.make_config("C3", n_chirps=64)
    rp, gp, bp = _params(scn)
    info = sar.sar_plan_geometry(rp, gp, bp)
    r = scn.radar
    mu = r.bandwidth_hz / r.chirp_s
    assert math.isclose(info.chirp_rate_hz_per_s, mu, rel_tol=1e-15)
    # a1: bins per metre of two-way path = mu N / (c fs) = B Z / c (Z = N/Ns)
    assert math.isclose(info.a1_bins_per_m, r.bandwidth_hz * 8 / sarsim.C_LIGHT, rel_tol=1e-12)
    assert abs(info.a1_bins_per_m - 24.84) < 0.01
    assert abs(info.c2_cycles_per_m - 255.51) < 0.01
    # crop covers every (pixel, antenna) two-way path: brute force over grid corners + track
    g = scn.grid
    corners = np.array([[g.x0, g.y0, 0], [g.x0 + (g.nx - 1) * g.dx, g.y0, 0],
                        [g.x0, g.y0 + (g.ny - 1) * g.dy, 0],
                        [g.x0 + (g.nx - 1) * g.dx, g.y0 + (g.ny - 1) * g.dy, 0]])
    d = 2 * np.linalg.norm(corners[:, None, :] - scn.tx[None, :, :], axis=2)
    # nearest pixel to the track: y = 1 row, x across the aperture
    xs = np.linspace(g.x0, g.x0 + (g.nx - 1) * g.dx, 3001)
    near = np.stack([xs, np.full_like(xs, g.y0), 0 * xs], 1)
    dn = 2 * np.linalg.norm(near[:, None, :] - scn.tx[None, ::8, :], axis=2)
    kmin = info.a1_bins_per_m * dn.min()
    kmax = info.a1_bins_per_m * d.max()
    assert info.k_lo <= math.floor(kmin) and info.k_lo + info.n_bins - 1 >= math.floor(kmax) + 1
    assert info.k_lo + info.n_bins - 1 <= r.fft_len // 2 + 1 and info.n_bins % 2 == 0
    # roughly the 1750 bins SURVEY 8(d) estimates for C3
    assert 1500 < info.n_bins < 1900
    assert info.tile_x == 32 and info.tile_y == 32
    rho = math.hypot(15.5 * g.dx, 15.5 * g.dy)
    assert info.window_bins == math.ceil(4 * info.a1_bins_per_m * rho * (1 + 1e-9)) + 4
    assert info.updates_per_image == g.nx * g.ny * 64


def test_plan_geometry_rejects_bad_parameters(lib):
    scn = sarsim.make_config("C1")
    bad = [dict(fft_len=1000), dict(fft_len=128), dict(n_samples=1), dict(sample_rate_hz=1e6),
           dict(pri_s=1e-6), dict(n_rx=0), dict(range_window=3), dict(bandwidth_hz=-1.0),
           dict(doppler_max_bins=-1.0), dict(fft_len=32768)]
    for kw in bad:
        rp, gp, bp = _params(scn, **kw)
        with pytest.raises(sar.SarError) as e:
            sar.sar_plan_geometry(rp, gp, bp)
        assert e.value.status == 1, kw
        assert sar.load().sar_last_error()
    rp, gp, bp = _params(scn)
    gp.dx = 0.0
    with pytest.raises(sar.SarError):
        sar.sar_plan_geometry(rp, gp, bp)
    rp, gp, bp = _params(scn)
    bp.lo[0], bp.hi[0] = 1.0, -1.0
    with pytest.raises(sar.SarError):
        sar.sar_plan_geometry(rp, gp, bp)


def test_paper_grid_window_and_stage_sizes(lib):
    """C0: the paper's 1201^2 grid at 2.5 cm: wider tiles in metres, wider windows."""
    scn = sarsim.make_config("C0", n_chirps=16)
    rp, gp, bp = _params(scn)
    info = sar.sar_plan_geometry(rp, gp, bp)
    assert info.updates_per_image == 1201 * 1201 * 16
    assert 50 < info.window_bins < 70
    assert info.chirps_per_stage >= 1


def test_plan_create_without_gpu_reports_device_error(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    scn = sarsim.make_config("C1")
    rp, gp, bp = _params(scn)
    with pytest.raises(sar.SarError) as e:
        sar.sar_plan_create(rp, gp, bp, 0)
    assert e.value.status in (3, 5)


def test_bp_kernel_sass_uses_bulk_copies_packed_fp32_and_mbarriers():
    """Blackwell-native evidence in the built library: the BP producer's 1-D bulk copies (TMA
    engine, UBLKCP), the consumers' packed fp32 pairs (FFMA2), MUFU rsqrt/sin/cos and the
    mbarrier ring (SYNCS) are all in bp_kernel's SASS."""
    _build.build()
    sass = subprocess.run(["cuobjdump", "-sass", _build.LIB], capture_output=True, text=True).stdout
    funcs = sass.split("Function : ")
    bp = "".join(f for f in funcs if f.startswith("_ZN3sar") and "bp_kernel_mono" in f.split("\n", 1)[0])
    assert bp, "bp_kernel_mono not found in libsar.so"
    for mnemonic in ("UBLKCP", "FFMA2", "MUFU.RSQ", "MUFU.SIN", "MUFU.COS", "SYNCS.ARRIVE", "SYNCS.PHASECHK"):
        assert mnemonic in bp, mnemonic


def test_rc_register_path_sass_uses_bulk_copy_ring():
    """The register-path range compression's raw-row ring: 1-D bulk copies (UBLKCP) completing
    on mbarriers (SYNCS), warp-level exchanges only inside the FFT (one block barrier per
    row pair before and after the epilogue)."""
    _build.build()
    sass = subprocess.run(["cuobjdump", "-sass", _build.LIB], capture_output=True, text=True).stdout
    funcs = sass.split("Function : ")
    ring = [f for f in funcs if f.startswith("_ZN3sar") and "rc_kernel_warpILi512ELi8ELi4E" in f.split("\n", 1)[0]]
    assert ring, "rc_kernel_warp<512, 8, 4> not found in libsar.so"
    body = ring[0]
    for mnemonic in ("UBLKCP", "SYNCS.PHASECHK", "LDS.64", "STS.64"):
        assert mnemonic in body, mnemonic
    assert body.count("BAR.SYNC") <= 3


def test_binding_fails_loudly_without_the_library(tmp_path):
    """No CPU fallback: with libsar.so absent the binding raises on first use."""
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2306_09784_b200 import sar\n"
            "try:\n    sar.load()\nexcept ImportError as e:\n    print('raised', e)\n") % ROOT
    env = dict(os.environ, SAR_LIB=str(tmp_path / "libsar.so"))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0 and "raised" in out.stdout and "missing" in out.stdout
