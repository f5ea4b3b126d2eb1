"""Small launches of every kernel family, run against the bounds-check build (-DSAR_DEBUG_CHECKS,
tools/variants/libsar_check.so via SAR_LIB): range compression (register and classic paths), plain
BP (unsplit and chirp-split with the split-sum kernel), near-field tiles (side stream), bistatic,
Doppler (incl. a table exceeding its declared bound: clamped), polar + resampling (incl. an antenna
outside the declared box: clamped into it), the split-publish scatter, tile shards, sar_image_sum.
(tools/variants/libsar_check.so was the tuning-build name; __graft_entry__.build() makes
paper_2306_09784_b200/libsar_check.so.)
compute-sanitizer is closed on this GPU pool, so the kernels count their own violations (window
index outside the item's entries, workspace plane out of range, bulk copy outside its row) and every
case also checks its image for consistency.

usage: SAR_LIB=paper_2306_09784_b200/libsar_check.so python tools/check_cases.py [case ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import sarsim
from paper_2306_09784_b200 import sar

dev = torch.device("cuda:0")


def _plan(scn, **kw):
    lo, hi = scn.antenna_box(1e-3)
    return sar.Plan(scn.radar, scn.grid, scn.n_chirps, scn.n_rx, (lo, hi), **kw)


def case_plain():
    scn = sarsim.small_config(n_chirps=64, ns=128, nx=70, ny=45, seed=3)   # unsplit, 2 x 3 tiles
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    p = _plan(scn)
    tx = torch.as_tensor(scn.tx, device=dev)
    prof = p.range_compress(raw)
    img = p.backproject(prof, tx)
    rows = p.backproject(prof, tx, row0=13, nrow=20)
    torch.cuda.synchronize()
    assert torch.equal(rows, img[13:33])
    p.close()


def case_split():
    scn = sarsim.small_config(n_chirps=2048, ns=128, nx=40, ny=33, seed=4, curved=True)   # chirp-split
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    p = _plan(scn)
    tx = torch.as_tensor(scn.tx, device=dev)
    prof = p.range_compress(raw)
    img = p.backproject(prof, tx)
    acc = img.clone()
    p.backproject(prof, tx, out=acc, accumulate=True)
    tiled = torch.zeros_like(img)
    p.backproject_tiles(prof, tx, 1, 2, out=tiled)
    p.backproject_tiles(prof, tx, 0, 1, out=tiled)
    p.backproject_tiles(prof, tx, 3, 1, out=tiled)
    torch.cuda.synchronize()
    assert float((acc - 2 * img).abs().max() / img.abs().max()) < 1e-6
    assert float((tiled - img).abs().max() / img.abs().max()) < 1e-6
    p.close()


def case_near_bistatic():
    # the track runs through the grid (near-field tiles on the side stream), 3 RX
    scn = sarsim.small_config(n_chirps=96, ns=128, nx=64, ny=64, seed=5, n_rx=3, grid_dx=0.01)
    g = scn.grid
    scn.grid = sarsim.Grid(g.x0, -0.2, g.z0, g.dx, g.dy, g.nx, g.ny)
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    p = _plan(scn)
    tx = torch.as_tensor(scn.tx, device=dev)
    rx = torch.as_tensor(scn.rx, device=dev).contiguous()
    prof = p.range_compress(raw)
    img = p.backproject(prof, tx, rx)
    torch.cuda.synchronize()
    assert torch.isfinite(torch.view_as_real(img)).all()
    p.close()


def case_doppler():
    scn = sarsim.small_config(n_chirps=64, ns=128, nx=40, ny=40, seed=6)
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    q = scn.tx.mean(0)
    v = np.array([8.0, 0.0, 0.0])
    dop = sar.doppler_table(scn.radar, scn.grid, q, v)
    bound = sar.doppler_bound_bins(scn.radar, v)
    lo, hi = scn.antenna_box(1e-3)
    p = sar.Plan(scn.radar, scn.grid, scn.n_chirps, 1, (lo, hi), doppler_max_bins=bound)
    tx = torch.as_tensor(scn.tx, device=dev)
    prof = p.range_compress(raw)
    img = p.backproject(prof, tx, doppler=dop)
    torch.cuda.synchronize()
    assert torch.isfinite(torch.view_as_real(img)).all()
    p.close()


def case_polar():
    scn = sarsim.polar_small_config(n_chirps=64, ns=256, n_th=70, n_r=40, seed=7)
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    p = _plan(scn)
    tx = torch.as_tensor(scn.tx, device=dev)
    prof = p.range_compress(raw)
    img = p.backproject(prof, tx)
    cart = sarsim.Grid(-0.5, 1.0, 0.0, 0.02, 0.02, 50, 40)
    out = sar.polar_to_cartesian(scn.grid, img, cart)
    torch.cuda.synchronize()
    assert torch.isfinite(torch.view_as_real(out)).all()
    p.close()


def case_scatter_split():
    scn = sarsim.small_config(n_chirps=4096, ns=128, nx=40, ny=24, seed=57)
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    p = _plan(scn)
    tx = torch.as_tensor(scn.tx, device=dev)
    prof = p.range_compress(raw)
    ref = p.backproject(prof, tx, row0=5, nrow=13)
    imgs = [torch.zeros((24, 40), dtype=torch.complex64, device=dev) for _ in range(2)]
    p.backproject_scatter(prof, tx, [im.data_ptr() for im in imgs], row0=5, nrow=13)
    p.backproject_scatter_tiles(prof, tx, [im.data_ptr() for im in imgs], 0, 1)
    torch.cuda.synchronize()
    assert torch.equal(imgs[0][5:18, 32:], ref[:, 32:])
    p.close()


def case_rc_classic():
    os.environ["SAR_RC_CLASSIC"] = "1"
    try:
        scn = sarsim.small_config(n_chirps=33, ns=128, nx=16, ny=16, seed=8)
        raw = sarsim.simulate_raw(scn, device="cuda:0")
        p = _plan(scn)
        p.range_compress(raw)
        torch.cuda.synchronize()
        p.close()
    finally:
        del os.environ["SAR_RC_CLASSIC"]


def case_sum():
    parts = torch.view_as_complex(torch.randn((3, 17, 33, 2), device=dev).contiguous())
    out = sar.image_sum(parts)
    torch.cuda.synchronize()
    assert torch.allclose(out, parts.sum(0), atol=1e-5)


def case_doppler_over_bound():
    """A Doppler table 3x its declared bound: clamped per pixel, the window index stays in range."""
    scn = sarsim.small_config(n_chirps=64, ns=128, nx=40, ny=40, seed=9)
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    lo, hi = scn.antenna_box(1e-3)
    p = sar.Plan(scn.radar, scn.grid, scn.n_chirps, 1, (lo, hi), doppler_max_bins=0.5)
    dop = torch.full((40, 40), 1.5, dtype=torch.float32, device=dev)
    tx = torch.as_tensor(scn.tx, device=dev)
    img = p.backproject(p.range_compress(raw), tx, doppler=dop)
    torch.cuda.synchronize()
    assert torch.isfinite(torch.view_as_real(img)).all()
    p.close()


def case_polar_antenna_outside_box():
    """Positions outside the declared box would break the polar window bound: a polar plan clamps
    them into the box, so every window read stays in range (values are wrong, by contract)."""
    scn = sarsim.polar_small_config(n_chirps=64, ns=256, n_th=70, n_r=40, seed=10)
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    lo, hi = scn.antenna_box(1e-3)
    p = sar.Plan(scn.radar, scn.grid, scn.n_chirps, scn.n_rx, (lo, hi))
    tx = torch.as_tensor(scn.tx, device=dev).clone()
    tx[:, 0] += 3.0   # 3 m beside the declared box
    img = p.backproject(p.range_compress(raw), tx)
    torch.cuda.synchronize()
    assert torch.isfinite(torch.view_as_real(img)).all()
    p.close()


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}
# cases whose inputs break the declared contract: the window-index and bulk-copy counters may count
# there (wrong values by contract); reads outside the allocation never
CONTRACT_BROKEN = {"polar_antenna_outside_box"}


def violations(reset=True):
    import ctypes

    lib = sar.load()
    out = []
    for fam in ("plain", "scatter"):
        f = getattr(lib, f"sar_debug_violations_{fam}", None)
        if f is None:
            raise SystemExit("not a bounds-check build: SAR_LIB=paper_2306_09784_b200/libsar_check.so")
        buf = (ctypes.c_ulonglong * 4)()
        f(buf, int(reset))
        out.append(list(buf))
    return [a + b for a, b in zip(*out)]


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    bad = 0
    for n in names:
        CASES[n]()
        torch.cuda.synchronize()
        v = violations()
        allowed = n in CONTRACT_BROKEN
        ok = v[1] == 0 and v[3] == 0 and (allowed or (v[0] == 0 and v[2] == 0))
        bad += not ok
        print(f"case {n}: violations window={v[0]} ws_plane={v[1]} bulk_copy={v[2]} smem_bounds={v[3]} -> "
              f"{'ok' if ok else 'FAIL'}",
              flush=True)
    sys.exit(1 if bad else 0)
