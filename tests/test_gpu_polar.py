"""GPU parity on the polar reconstruction grid (Measure E; NEXT-1): the BP
kernel on polar pixels and the polar -> Cartesian resampling kernel, through the C ABI,
against the fp64 oracle on the same seeded inputs (bar: peak indices equal and
max|gpu - ref| / max|ref| <= 1e-3)."""
import numpy as np
import pytest

import oracle
import sarsim
from sarsim import Grid, PolarGrid

from .helpers import REL_TOL, gpu_image, oracle_image, rel_err
from .helpers import oracle_profiles as oracle_profiles_crop

pytestmark = pytest.mark.gpu


def _scene(kind):
    if kind == "straight":
        return sarsim.polar_small_config(n_chirps=96, n_th=77, n_r=45, seed=41)
    if kind == "curved_bistatic":
        return sarsim.polar_small_config(n_chirps=64, n_th=50, n_r=33, n_rx=3, curved=True, seed=42)
    if kind == "wide_sector":     # bearings across +-1 rad: tiles sheared far from axis-aligned
        return sarsim.polar_small_config(n_chirps=64, n_th=100, n_r=20, th0=-1.0, dth=0.02, r0=3.0,
                                         dr=0.05, seed=43)
    if kind == "near_field":      # polar centre on the track: innermost ring 2 cm from antennas
        return sarsim.polar_small_config(n_chirps=48, n_th=64, n_r=40, r0=0.02, dr=0.03, th0=-0.5,
                                         dth=0.016, seed=44)
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["straight", "curved_bistatic", "wide_sector", "near_field"])
def test_polar_bp_full_image_parity(cuda_lib, kind):
    scn = _scene(kind)
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    got = gpu_image(scn, raw).cpu().numpy().reshape(-1)
    ref = oracle_image(scn, raw.cpu().numpy())
    assert np.argmax(np.abs(got)) == np.argmax(np.abs(ref))
    assert rel_err(got, ref) <= REL_TOL


def test_polar_row_shards_equal_unsharded(cuda_lib):
    import torch

    scn = _scene("straight")
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    full, prof, plan = gpu_image(scn, raw, return_prof=True)
    tx = torch.as_tensor(scn.tx, device="cuda:0")
    ty = plan.info.tile_y
    parts = [plan.backproject(prof, tx, row0=r0, nrow=min(ty, scn.grid.n_r - r0))
             for r0 in range(0, scn.grid.n_r, ty)]
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts), full)      # tile-aligned rows: same anchors, same sums
    plan.close()


@pytest.mark.parametrize("th0", [-0.7, 2.5, -0.7 + 2 * np.pi])
def test_polar_to_cartesian_kernel_matches_oracle(cuda_lib, th0):
    """The resampling kernel against the oracle, also for a sector crossing +-pi (centred on -y)
    and for th0 given in the next period."""
    import torch

    pg = PolarGrid(0.1, -0.3, 0.0, 2.0, 0.03, th0, 0.012, 117, 61)
    rng = np.random.default_rng(7)
    img = (rng.standard_normal((pg.n_r, pg.n_th)) + 1j * rng.standard_normal((pg.n_r, pg.n_th)))
    img = img.astype(np.complex64)
    # a grid around the sector: ahead of the centre (+y) or behind it (-y)
    ahead = np.cos(th0 + 0.5 * (pg.n_th - 1) * pg.dth) > 0
    cart = Grid(-2.0, 0.5, 0.0, 0.021, 0.019, 203, 197) if ahead else Grid(-2.0, -4.5, 0.0, 0.021, 0.019, 203, 197)
    got = cuda_lib.polar_to_cartesian(pg, torch.as_tensor(img, device="cuda:0"), cart)
    torch.cuda.synchronize()
    got = got.cpu().numpy()
    ref = oracle.polar_to_cartesian(pg, img.astype(np.complex128), cart)
    inside = ref != 0
    assert inside.sum() > 5000 and (~inside).sum() > 5000
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()
    assert np.all(got[~inside] == 0)


def test_polar_image_resampled_peaks_where_the_cartesian_image_does(cuda_lib):
    """The polar image of a point target, resampled, peaks within one Cartesian pixel of
    the Cartesian image's peak, and the two agree there to interpolation accuracy."""
    import torch

    scn = sarsim.polar_small_config(n_chirps=96, n_th=60, n_r=40, dth=0.02, dr=0.04, th0=-0.6, seed=45)
    k = 0
    raw = sarsim.simulate_raw(scn, device="cuda:0", targets=scn.targets[k:k + 1], amps=scn.amps[k:k + 1])
    pimg = gpu_image(scn, raw)
    tgt = scn.targets[k]
    cart = Grid(tgt[0] - 0.2, tgt[1] - 0.2, 0.0, 0.01, 0.01, 41, 41)
    cscn = sarsim.Scenario("cart", scn.radar, cart, scn.tx, scn.rx, scn.targets, scn.amps, scn.isolated,
                           scn.wsar)
    cimg = gpu_image(cscn, raw).cpu().numpy()
    rs = cuda_lib.polar_to_cartesian(scn.grid, pimg, cart)
    torch.cuda.synchronize()
    rs = rs.cpu().numpy()
    pc = np.unravel_index(np.argmax(np.abs(cimg)), cimg.shape)
    pr = np.unravel_index(np.argmax(np.abs(rs)), rs.shape)
    assert pc == (20, 20)
    assert abs(pr[0] - pc[0]) <= 1 and abs(pr[1] - pc[1]) <= 1
    assert abs(abs(rs[pc]) - abs(cimg[pc])) < 0.1 * abs(cimg[pc])


def test_C6p_full_size_sampled_parity(cuda_lib):
    """The bench's Measure E workload (C6p: 520 x 315 polar pixels, 1024 chirps x 8 RX) in the
    bench's launch configuration against the oracle on a strided sample plus windows around the
    GPU's strongest pixels; then the resampling kernel on the same image."""
    import torch

    scn = sarsim.make_config("C6p")
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    img, prof, plan = gpu_image(scn, raw, return_prof=True)
    g = scn.grid
    a = np.abs(img.cpu().numpy())
    js, iis = np.arange(0, g.n_r, 23), np.arange(0, g.n_th, 7)
    pts = [np.stack(np.meshgrid(js, iis, indexing="ij"), -1).reshape(-1, 2)]
    for f in np.argsort(a.reshape(-1))[::-1][:16]:
        j, i = np.unravel_index(f, a.shape)
        jj, ii = np.meshgrid(np.arange(j - 2, j + 3), np.arange(i - 2, i + 3), indexing="ij")
        w = np.stack([jj, ii], -1).reshape(-1, 2)
        pts.append(w[(w[:, 0] >= 0) & (w[:, 0] < g.n_r) & (w[:, 1] >= 0) & (w[:, 1] < g.n_th)])
    idx = np.unique(np.concatenate(pts), axis=0)
    ref_prof = oracle_profiles_crop(scn, raw.cpu().numpy(), plan.k_lo, plan.n_bins)
    ref = oracle.backproject(ref_prof, plan.k_lo, scn.radar, scn.tx, scn.rx, g.pixel_list(idx))
    got = img.cpu().numpy()[idx[:, 0], idx[:, 1]]
    assert rel_err(got, ref) <= REL_TOL
    k = int(np.argmax(np.abs(ref)))
    assert tuple(idx[k]) == np.unravel_index(np.argmax(a), a.shape)
    cart = sarsim.make_config("C0", n_chirps=1).grid
    rs = cuda_lib.polar_to_cartesian(g, img, cart)
    torch.cuda.synchronize()
    sub = (slice(0, None, 37), slice(0, None, 41))
    ref_rs = oracle.polar_to_cartesian(g, img.cpu().numpy().astype(np.complex128),
                                       Grid(cart.x0, cart.y0, 0.0, cart.dx * 41, cart.dy * 37,
                                            len(range(0, cart.nx, 41)), len(range(0, cart.ny, 37))))
    assert np.abs(rs.cpu().numpy()[sub] - ref_rs).max() <= 1e-5 * np.abs(ref_rs).max()
    plan.close()


def test_polar_doppler_table_and_bp_match_oracle(cuda_lib):
    """Measure D on a Measure E grid: the polar Doppler table kernel against the oracle's table
    on the polar pixels, and the Doppler-corrected polar BP of a Doppler-aware simulation
    against the oracle."""
    import torch

    scn = sarsim.polar_small_config(n_chirps=96, n_th=60, n_r=32, seed=46)
    # a moving platform: 9 m/s at the chirp period
    scn.tx = sarsim.straight_track(scn.n_chirps, 9.0 * scn.radar.pri_s)
    q_ref = scn.tx.mean(0)
    v_avg = sarsim.track_velocity(scn).mean(0)
    got = cuda_lib.doppler_table(scn.radar, scn.grid, q_ref, v_avg)
    torch.cuda.synchronize()
    ref = oracle.doppler_table(scn.radar, scn.grid.pixels(), q_ref, v_avg).reshape(scn.grid.n_r, scn.grid.n_th)
    assert np.abs(got.cpu().numpy() - ref).max() < 1e-5 * max(1.0, np.abs(ref).max())
    raw = sarsim.simulate_raw(scn, device="cuda:0", doppler=True)
    dmax = float(np.abs(ref).max()) + 0.5
    img = gpu_image(scn, raw, doppler=ref.astype(np.float32), dop_max=dmax).cpu().numpy().reshape(-1)
    oref = oracle_image(scn, raw.cpu().numpy(), doppler=ref.reshape(-1))
    assert np.argmax(np.abs(img)) == np.argmax(np.abs(oref))
    assert rel_err(img, oref) <= REL_TOL
