"""GPU parity (-m gpu): the CUDA path through the C ABI against the fp64 oracle on the same
seeded inputs.  Bar (north star): peak pixel indices equal and
max|img_gpu - img_ref| / max|img_ref| <= 1e-3; profiles within 1e-5 of max|ref|."""
import os

import numpy as np
import pytest

import oracle
import sarsim
from sarsim import C_LIGHT, Grid, Scenario

from .helpers import REL_TOL, c6_indices, gpu_image, oracle_image, oracle_profiles, rel_err, sample_indices

pytestmark = pytest.mark.gpu


def _raw(scn):
    import torch

    return sarsim.simulate_raw(scn, device="cuda:0")


# ----------------------------------------------------------------------------- range compression
@pytest.mark.parametrize("path", ["register", "classic"])
@pytest.mark.parametrize("cfg", ["C1", "small_hann", "small_rect_odd", "C2_256", "ns500_z1", "ns200_z2",
                                 "ns300_z16"])
def test_rc_profiles_match_oracle(cuda_lib, cfg, path, monkeypatch):
    """Both range-compression kernels (the register path: Zp = N/L warp transforms of length
    L = 256/512; the classic shared-memory FFT, forced by SAR_RC_CLASSIC=1) on every
    transform shape class: Z = 1, 2, 4, 8, 16, 32, odd log2 N, ragged Ns, odd row counts."""
    if path == "classic":
        monkeypatch.setenv("SAR_RC_CLASSIC", "1")
    else:
        monkeypatch.delenv("SAR_RC_CLASSIC", raising=False)
    if cfg.startswith("ns"):
        ns, nfft = {"ns500_z1": (500, 512), "ns200_z2": (200, 512), "ns300_z16": (300, 8192)}[cfg]
        scn = sarsim.small_config(n_chirps=9, ns=128, n_rx=1, seed=7, noise_sigma=0.1)
        scn.radar = sarsim.Radar(n_samples=ns, fft_len=nfft, range_window=1)
    elif cfg == "C1":
        scn = sarsim.make_config("C1", wsar="hann")
    elif cfg == "small_hann":
        scn = sarsim.small_config(n_chirps=37, ns=128, n_rx=3, seed=5, noise_sigma=0.1)
        scn.wsar = np.linspace(0.2, 1.0, 37).astype(np.float32)
    elif cfg == "small_rect_odd":
        scn = sarsim.small_config(n_chirps=5, ns=64, seed=6)
        scn.radar = sarsim.Radar(n_samples=64, fft_len=2048, range_window=0)   # Z = 32, odd log2
    else:
        scn = sarsim.make_config("C2", n_chirps=256)
    raw = _raw(scn)
    img, prof, plan = gpu_image(scn, raw, return_prof=True)
    ref = oracle_profiles(scn, raw.cpu().numpy(), plan.k_lo, plan.n_bins)
    got = prof.cpu().numpy()
    err = np.abs(got - ref).max() / np.abs(ref).max()
    plan.close()
    assert err < 1e-5, err


def test_rc_chirp_shards_write_only_their_rows(cuda_lib):
    import torch

    scn = sarsim.small_config(n_chirps=20, ns=128, n_rx=2, seed=8)
    raw = _raw(scn)
    lo, hi = scn.antenna_box(1e-3)
    plan = cuda_lib.Plan(scn.radar, scn.grid, 20, 2, (lo, hi))
    full = plan.range_compress(raw)
    part = torch.full_like(full, complex(7.0, 7.0))
    plan.range_compress(raw, chirp0=5, nchirp=9, out=part)
    torch.cuda.synchronize()
    assert torch.equal(part[5:14], full[5:14])
    assert torch.all(part[:5] == complex(7.0, 7.0)) and torch.all(part[14:] == complex(7.0, 7.0))
    plan.close()


# ----------------------------------------------------------------------------- full chain, small
def test_C1_full_image_parity(cuda_lib):
    scn = sarsim.make_config("C1")
    raw = _raw(scn)
    got = gpu_image(scn, raw).cpu().numpy().reshape(-1)
    ref = oracle_image(scn, raw.cpu().numpy())
    assert np.argmax(np.abs(got)) == np.argmax(np.abs(ref)) == 32 * 64 + 32
    assert rel_err(got, ref) <= REL_TOL
    # phase at the peak: arg P(p*) = arg a (A2) to 1e-3 rad
    assert abs(np.angle(got[32 * 64 + 32])) < 1e-3


@pytest.mark.parametrize("kind", ["ragged_straight", "curved_bistatic", "curved_hann", "fine_grid"])
def test_small_scenes_full_image_parity(cuda_lib, kind):
    if kind == "ragged_straight":
        scn = sarsim.small_config(n_chirps=96, ns=256, nx=77, ny=45, seed=21)
    elif kind == "curved_bistatic":
        scn = sarsim.small_config(n_chirps=64, ns=256, nx=50, ny=33, n_rx=3, curved=True, seed=22)
    elif kind == "curved_hann":
        scn = sarsim.small_config(n_chirps=128, ns=256, nx=64, ny=64, curved=True, seed=23, noise_sigma=0.2)
        u = np.arange(128) / 127.0
        scn.wsar = (0.5 - 0.5 * np.cos(2 * np.pi * u)).astype(np.float32)
    else:
        scn = sarsim.small_config(n_chirps=64, ns=256, nx=70, ny=40, seed=24, grid_dx=0.004)
    raw = _raw(scn)
    got = gpu_image(scn, raw).cpu().numpy().reshape(-1)
    ref = oracle_image(scn, raw.cpu().numpy())
    assert np.argmax(np.abs(got)) == np.argmax(np.abs(ref))
    assert rel_err(got, ref) <= REL_TOL
    # local peaks around every isolated target agree wherever the oracle's peak is
    # unambiguous (best/second > 1 + 4e-3, reading A15: ties cannot flip under 1e-3)
    G = np.abs(got.reshape(scn.grid.ny, scn.grid.nx))
    R = np.abs(ref.reshape(scn.grid.ny, scn.grid.nx))
    for (j, i) in scn.isolated:
        sl = (slice(max(0, j - 2), j + 3), slice(max(0, i - 2), i + 3))
        r = np.sort(R[sl].ravel())
        if r[-1] > (1 + 4e-3) * r[-2]:
            assert np.argmax(G[sl]) == np.argmax(R[sl])


# ----------------------------------------------------------------------------- closed forms on GPU
def test_flat_profile_exact_coherent_sum_gpu(cuda_lib):
    """T4 on the GPU BP alone: X_m[k] = a exp(-j 2 pi f0 d_m(p*)/c) for all k -> P(p*) = a M."""
    import torch

    r = sarsim.Radar(n_samples=256, fft_len=2048)
    M = 300
    tx = sarsim.curved_track(M, r.pri_s, 6, 9, 20.0)
    grid = Grid(-0.5, 20.0, 0.0, 0.01, 0.01, 64, 40)
    pj, pi_ = 17, 41
    p = np.array([grid.x0 + pi_ * grid.dx, grid.y0 + pj * grid.dy, 0.0])
    d = 2 * np.linalg.norm(tx - p, axis=1)
    a = 0.8 * np.exp(0.3j)
    lo, hi = tx.min(0) - 1e-3, tx.max(0) + 1e-3
    plan = cuda_lib.Plan(r, grid, M, 1, (lo, hi))
    row = a * np.exp(-2j * np.pi * r.f0_hz * d / C_LIGHT)
    prof = torch.as_tensor(np.repeat(row[:, None, None], plan.n_bins, axis=2).astype(np.complex64), device="cuda:0")
    img = plan.backproject(prof, torch.as_tensor(tx, device="cuda:0"))
    torch.cuda.synchronize()
    v = complex(img[pj, pi_].item())
    plan.close()
    # the only error left is fp32 rounding of the flat row itself (1e-7) and the range form
    assert abs(v - a * M) < 1e-5 * M, (v, a * M)


def test_translation_invariance_gpu(cuda_lib):
    """T7: a 1 km shift of track, grid and scene changes nothing (fp32 accuracy form)."""
    scn = sarsim.small_config(n_chirps=128, ns=256, nx=48, ny=40, seed=31)
    raw = _raw(scn)
    ref = oracle_image(scn, raw.cpu().numpy())
    sh = np.array([1000.0, 1000.0, 0.0])
    g = scn.grid
    scn2 = Scenario("shift", scn.radar, Grid(g.x0 + 1000, g.y0 + 1000, 0.0, g.dx, g.dy, g.nx, g.ny),
                    scn.tx + sh, None, scn.targets + sh, scn.amps, scn.isolated, scn.wsar)
    got = gpu_image(scn2, raw).cpu().numpy().reshape(-1)
    assert rel_err(got, ref) <= REL_TOL
    assert np.argmax(np.abs(got)) == np.argmax(np.abs(ref))


@pytest.mark.parametrize("n_rx", [1, 2])
def test_chirp_permutation_gpu(cuda_lib, n_rx, monkeypatch):
    """T6 on the GPU.  With one rsqrt leg per chirp (SAR_BP_DERIVE=0) the image is order-invariant
    to fp32 summation order (1e-5).  By default, groups of consecutive chirps whose positions are
    close take their legs from the group base by the series (reading A22); a permutation breaks
    the groups up, so the two images differ by the series' rounding (<= 1e-8 m per leg, checked
    at 1e-4) and both meet the oracle bar."""
    scn = sarsim.small_config(n_chirps=96, ns=256, nx=40, ny=30, curved=True, n_rx=n_rx, seed=32)
    raw = _raw(scn)
    perm = np.random.default_rng(2).permutation(96)
    rx = None if scn.rx is None else scn.rx[perm]
    scn2 = Scenario("perm", scn.radar, scn.grid, scn.tx[perm], rx, scn.targets, scn.amps, scn.isolated,
                    scn.wsar[perm])
    raw2 = raw[perm.tolist()].contiguous()
    a = gpu_image(scn, raw).cpu().numpy()
    b = gpu_image(scn2, raw2).cpu().numpy()
    ref = oracle_image(scn, raw.cpu().numpy()).reshape(a.shape)
    assert rel_err(b, a) < 1e-4
    assert rel_err(a, ref) <= REL_TOL and rel_err(b, ref) <= REL_TOL
    monkeypatch.setenv("SAR_BP_DERIVE", "0")
    a0 = gpu_image(scn, raw).cpu().numpy()
    b0 = gpu_image(scn2, raw2).cpu().numpy()
    assert rel_err(b0, a0) < 1e-5


def test_doppler_term_matches_oracle(cuda_lib):
    """Alg. 2 L8 f_doppler(p) (Measure D): per-pixel index shift, same on both sides."""
    scn = sarsim.small_config(n_chirps=64, ns=256, nx=40, ny=36, seed=33)
    g = scn.grid
    rng = np.random.default_rng(0)
    dop = rng.uniform(-0.6, 0.6, (g.ny, g.nx)).astype(np.float32)
    raw = _raw(scn)
    got = gpu_image(scn, raw, doppler=dop, dop_max=0.6).cpu().numpy().reshape(-1)
    ref = oracle_image(scn, raw.cpu().numpy(), doppler=dop.reshape(-1).astype(np.float64))
    assert rel_err(got, ref) <= REL_TOL


def test_doppler_table_kernel_matches_oracle(cuda_lib):
    import torch

    scn = sarsim.make_config("C2", n_chirps=64)
    g = sarsim.Grid(-15.0, 1.0, 0.0, 0.01, 0.01, 700, 300)
    q, v = np.array([0.3, -0.1, 0.2]), np.array([7.5, 0.4, 0.0])
    got = cuda_lib.doppler_table(scn.radar, g, q, v).cpu().numpy().reshape(-1)
    ref = oracle.doppler_table(scn.radar, g.pixels(), q, v)
    assert np.abs(got - ref).max() <= 1e-6 * np.abs(ref).max()
    assert np.abs(ref).max() <= cuda_lib.doppler_bound_bins(scn.radar, v)


def test_doppler_full_chain_matches_oracle(cuda_lib):
    """Moving-platform simulator (Alg. 1 L11 Doppler) + Measure D table from the GPU kernel +
    BP with f_doppler(p) (Alg. 2 L8) against the oracle with the oracle's table."""
    import torch

    r = sarsim.Radar(n_samples=256, fft_len=2048)
    M = 512
    tx = sarsim.straight_track(M, 9.0 * r.pri_s)
    grid = Grid(-1.0, 1.5, 0.0, 0.01, 0.01, 250, 180)
    tg = np.array([[-0.6, 2.1, 0.0], [0.35, 2.6, 0.0], [0.9, 3.1, 0.0]])
    scn = Scenario("dop", r, grid, tx, None, tg, np.array([1.0, 0.7j, -0.5]), np.zeros((0, 2), int),
                   np.ones(M, np.float32))
    raw = sarsim.simulate_raw(scn, device="cuda:0", doppler=True)
    q_ref, v_avg = tx.mean(0), sarsim.track_velocity(scn).mean(0)
    dmax = cuda_lib.doppler_bound_bins(r, v_avg)
    dop = cuda_lib.doppler_table(r, grid, q_ref, v_avg)
    got = gpu_image(scn, raw, doppler=dop, dop_max=dmax).cpu().numpy().reshape(-1)
    ref = oracle_image(scn, raw.cpu().numpy(), doppler=oracle.doppler_table(r, grid.pixels(), q_ref, v_avg))
    assert rel_err(got, ref) <= REL_TOL
    assert np.argmax(np.abs(got)) == np.argmax(np.abs(ref))
    # a row shard: its pair rows cover only the shard's own crop (Doppler margin included)
    part = gpu_image(scn, raw, doppler=dop, dop_max=dmax, row0=70, nrow=50).cpu().numpy()
    ref2 = ref.reshape(grid.ny, grid.nx)[70:120]
    assert np.abs(part - ref2).max() <= REL_TOL * np.abs(ref).max()
    assert rel_err(part, ref2) <= 2 * REL_TOL


def test_near_field_pixel_on_antenna(cuda_lib):
    """T9: a pixel coincident with an antenna phase centre stays finite and matches the oracle."""
    r = sarsim.Radar(n_samples=256, fft_len=2048)
    M = 32
    tx = sarsim.straight_track(M, r.wavelength_m / 4, y=1.0)
    grid = Grid(-0.3, 0.9, 0.0, 0.01, 0.01, 64, 48)      # contains the track
    tx[:, 0] = np.round((tx[:, 0] - grid.x0) / 0.01) * 0.01 + grid.x0  # antennas on pixel centres
    scn = Scenario("near", r, grid, tx, None, np.array([[0.05, 1.2, 0.0]]), np.array([1.0 + 0j]),
                   np.zeros((0, 2), int), np.ones(M, np.float32))
    raw = _raw(scn)
    got = gpu_image(scn, raw).cpu().numpy().reshape(-1)
    assert np.all(np.isfinite(got))
    ref = oracle_image(scn, raw.cpu().numpy())
    assert rel_err(got, ref) <= REL_TOL


# ----------------------------------------------------------------------------- shards and edges
def test_row_and_chirp_shards_equal_unsharded(cuda_lib):
    """T11: every pixel is computed in its absolute grid tile with the tile's own fp64 anchor,
    so ANY row shard and any tile shard reproduce the unsharded image bit for bit (these
    launches are unsplit: 200 (chirp, RX) items); chirp shards agree to fp32 summation order."""
    import torch

    scn = sarsim.small_config(n_chirps=100, ns=256, nx=70, ny=90, seed=41, n_rx=2)
    raw = _raw(scn)
    img, prof, plan = gpu_image(scn, raw, return_prof=True)
    tx = torch.as_tensor(scn.tx, device="cuda:0")
    rx = torch.as_tensor(scn.rx, device="cuda:0").contiguous()
    ty = plan.info.tile_y
    aligned = torch.cat([plan.backproject(prof, tx, rx, row0=r0, nrow=n) for r0, n in ((0, ty), (ty, 90 - ty))])
    rows = torch.cat([plan.backproject(prof, tx, rx, row0=r0, nrow=n) for r0, n in ((0, 23), (23, 40), (63, 27))])
    tiles_x, tiles_y = plan.tiles
    assert (tiles_x, tiles_y) == (-(-70 // 32), -(-90 // ty))
    sentinel = complex(5.0, -5.0)
    tiled = torch.full((90, 70), sentinel, dtype=torch.complex64, device="cuda:0")
    for t0, nt in ((0, 2), (2, 3), (5, 1), (6, tiles_x * tiles_y - 6)):
        plan.backproject_tiles(prof, tx, t0, nt, rx, out=tiled)
    one = torch.full((90, 70), sentinel, dtype=torch.complex64, device="cuda:0")
    plan.backproject_tiles(prof, tx, 4, 1, rx, out=one)   # tile (1, 1): only its pixels written
    acc = plan.backproject(prof, tx, rx, chirp0=0, nchirp=37)
    plan.backproject(prof, tx, rx, chirp0=37, nchirp=63, out=acc, accumulate=True)
    # chirp shards regroup the derived legs (reading A22): fp32 order + the series' rounding;
    # with one rsqrt leg per chirp, fp32 summation order only
    os.environ["SAR_BP_DERIVE"] = "0"
    try:
        full0 = plan.backproject(prof, tx, rx)
        acc0 = plan.backproject(prof, tx, rx, chirp0=0, nchirp=37)
        plan.backproject(prof, tx, rx, chirp0=37, nchirp=63, out=acc0, accumulate=True)
    finally:
        del os.environ["SAR_BP_DERIVE"]
    torch.cuda.synchronize()
    a = img.cpu().numpy()
    assert torch.equal(aligned, img)
    assert torch.equal(rows, img)
    assert torch.equal(tiled, img)
    mask = torch.zeros((90, 70), dtype=torch.bool, device="cuda:0")
    mask[ty:2 * ty, 32:64] = True
    assert torch.equal(one[mask], img[mask]) and torch.all(one[~mask] == sentinel)
    assert rel_err(acc.cpu().numpy(), a) < 1e-4
    assert rel_err(acc0.cpu().numpy(), full0.cpu().numpy()) < 1e-5
    # empty chirp shard: zeros (overwrite) / untouched (accumulate); empty row/tile shard: no-op
    z = plan.backproject(prof, tx, rx, chirp0=10, nchirp=0)
    keep = acc.clone()
    plan.backproject(prof, tx, rx, chirp0=10, nchirp=0, out=acc, accumulate=True)
    plan.backproject(prof, tx, rx, row0=5, nrow=0, out=acc[:0])
    plan.backproject_tiles(prof, tx, 3, 0, rx, out=acc)
    torch.cuda.synchronize()
    assert torch.all(z == 0) and torch.equal(acc, keep)
    with pytest.raises(cuda_lib.SarError):
        plan.backproject_tiles(prof, tx, tiles_x * tiles_y - 1, 2, rx, out=acc)
    plan.close()


def test_chirp_split_for_small_grids(cuda_lib):
    """A grid of few tiles and many chirps runs as several chirp chunks per tile, each storing a
    partial image into its own workspace plane; a second kernel adds the planes in chunk order.
    Overwrite and accumulate match the oracle; the image is bit-reproducible run to run, and
    row / tile shards (other chunkings) agree to fp32 summation order."""
    import torch

    scn = sarsim.small_config(n_chirps=2048, ns=256, nx=48, ny=40, seed=45, curved=True)
    raw = _raw(scn)
    img, prof, plan = gpu_image(scn, raw, return_prof=True)
    ref = oracle_image(scn, raw.cpu().numpy())
    assert rel_err(img.cpu().numpy().reshape(-1), ref) <= REL_TOL
    tx = torch.as_tensor(scn.tx, device="cuda:0")
    n0 = plan.launches
    again = plan.backproject(prof, tx)
    torch.cuda.synchronize()
    assert plan.launches - n0 == 3   # pair rows, chirp-split BP, split sum
    assert torch.equal(again, img)
    twice = img.clone()
    plan.backproject(prof, tx, out=twice, accumulate=True)
    rows = torch.cat([plan.backproject(prof, tx, row0=r0, nrow=n) for r0, n in ((0, 7), (7, 30), (37, 3))])
    tiled = torch.zeros_like(img)
    for t0, nt in ((0, 1), (1, 2), (3, 1)):
        plan.backproject_tiles(prof, tx, t0, nt, out=tiled)
    torch.cuda.synchronize()
    assert rel_err(twice.cpu().numpy(), 2 * img.cpu().numpy()) < 1e-6
    assert rel_err(rows.cpu().numpy(), img.cpu().numpy()) < 1e-6
    assert rel_err(tiled.cpu().numpy(), img.cpu().numpy()) < 1e-6
    plan.close()


@pytest.mark.parametrize("world", [2, 8])
def test_C3_rank_partitions_assemble_the_one_gpu_image(cuda_lib, world):
    """The bench's N-GPU decompositions of C3, run rank by rank on one GPU: the tile partition
    (fused-gather leg) and the tile-row partition (NCCL all-gather leg) assemble the 1-GPU image
    to fp32 chunk order; every pixel is computed with the unsharded tile anchor.  The launches split
    their chirps into different chunk counts (a shard fills the GPU with more chunks), so the
    per-pixel sums differ in the order the chunk partials are added: measured 1.0-1.1e-6 (three
    resident CTAs per SM), checked at 2e-6, well inside T11's 1e-5 (reading A18)."""
    import torch

    from paper_2306_09784_b200.dist import tile_partition, tile_row_partition

    scn = sarsim.make_config("C3")
    raw = _raw(scn)
    img, prof, plan = gpu_image(scn, raw, return_prof=True)
    tx = torch.as_tensor(scn.tx, device="cuda:0")
    g = scn.grid
    tiles_x, tiles_y = plan.tiles
    tiled = torch.zeros_like(img)
    for r in range(world):
        t0, nt = tile_partition(tiles_x * tiles_y, world, r)
        plan.backproject_tiles(prof, tx, t0, nt, out=tiled)
    parts = [tile_row_partition(tiles_y, plan.info.tile_y, g.ny, world, r) for r in range(world)]
    assert sum(n for _, n in parts) == g.ny and parts[0][0] == 0
    rows = torch.cat([plan.backproject(prof, tx, row0=r0, nrow=n) for r0, n in parts])
    torch.cuda.synchronize()
    ref = img.abs().max()
    e_t = float((tiled - img).abs().max() / ref)
    e_r = float((rows - img).abs().max() / ref)
    plan.close()
    assert e_t <= 2e-6 and e_r <= 2e-6, (e_t, e_r)


def test_one_pixel_grid_and_single_chirp(cuda_lib):
    scn = sarsim.small_config(n_chirps=1, ns=128, nx=1, ny=1, seed=42)
    raw = _raw(scn)
    got = gpu_image(scn, raw).cpu().numpy().reshape(-1)
    ref = oracle_image(scn, raw.cpu().numpy())
    assert abs(got[0] - ref[0]) <= REL_TOL * max(abs(ref[0]), 1e-30) + 1e-6


def test_error_codes(cuda_lib):
    import torch

    sar = cuda_lib
    scn = sarsim.small_config(n_chirps=8, ns=64, nx=16, ny=16, seed=43)
    lo, hi = scn.antenna_box(1e-3)
    plan = sar.Plan(scn.radar, scn.grid, 8, 1, (lo, hi))
    raw = _raw(scn)
    prof = plan.range_compress(raw)
    tx = torch.as_tensor(scn.tx, device="cuda:0")
    with pytest.raises(sar.SarError) as e:
        plan.backproject(prof, tx, chirp0=4, nchirp=5)
    assert e.value.status == 1
    with pytest.raises(sar.SarError):
        plan.backproject(prof, tx, row0=10, nrow=7)
    with pytest.raises(sar.SarError):
        sar.sar_backproject(plan.handle, prof.data_ptr(), None, None, None, 0, 8, 0, 16, prof.data_ptr())
    with pytest.raises(sar.SarError):   # Doppler array without a declared bound
        plan.backproject(prof, tx, doppler=torch.zeros((16, 16), device="cuda:0"))
    # coverage: a TX position outside the declared box
    bad = scn.tx.copy()
    bad[3, 1] += 5.0
    with pytest.raises(sar.SarError) as e:
        plan.form_image(raw.cpu().contiguous(), torch.as_tensor(bad))
    assert e.value.status == 2
    plan.close()


def test_form_image_host_buffers_equal_device_path(cuda_lib):
    import torch

    scn = sarsim.small_config(n_chirps=64, ns=256, nx=40, ny=33, seed=44, n_rx=2)
    raw = _raw(scn)
    img, prof, plan = gpu_image(scn, raw, return_prof=True)
    raw_h = raw.cpu().pin_memory()
    out = plan.form_image(raw_h, torch.as_tensor(scn.tx).pin_memory(), torch.as_tensor(scn.rx).contiguous(),
                          torch.as_tensor(scn.wsar))
    torch.cuda.synchronize()
    assert torch.equal(out, img.cpu())
    assert plan.launches >= 4
    plan.close()


@pytest.mark.parametrize("cfg,rows", [("C3", (0, 3000)), ("C3", (96, 2000)), ("C2", (100, 700))])
def test_form_image_direct_host_stores_equal_device_path(cuda_lib, cfg, rows):
    """Shards that fill the GPU without a chirp split and a pinned host image take the fused
    readback (the BP epilogue stores into mapped host memory; pinned raw samples are read by
    the range compression in place); smaller shards and pageable images take the copy path.
    The copy path equals sar_backproject bit for bit; the direct path (unsplit when that fills
    8 waves) and the scatter into a device image differ from it only by the fp32 order of the
    chirp-chunk sums (32-wave split)."""
    import torch

    scn = sarsim.make_config(cfg, n_chirps=512)
    raw = _raw(scn)
    row0, nrow = rows
    lo, hi = scn.antenna_box(1e-3)
    plan = cuda_lib.Plan(scn.radar, scn.grid, scn.n_chirps, 1, (lo, hi))
    tx = torch.as_tensor(scn.tx, device="cuda:0")
    prof = plan.range_compress(raw)
    ref = plan.backproject(prof, tx, row0=row0, nrow=nrow).cpu()
    full = torch.zeros((scn.grid.ny, scn.grid.nx), dtype=torch.complex64, device="cuda:0")
    plan.backproject_scatter(prof, tx, [full.data_ptr()], row0=row0, nrow=nrow)
    unsplit = full[row0:row0 + nrow].cpu()
    raw_h, tx_h = raw.cpu().pin_memory(), torch.as_tensor(scn.tx).pin_memory()
    pinned = torch.full((nrow, scn.grid.nx), complex(5.0, 5.0), dtype=torch.complex64).pin_memory()
    out = plan.form_image(raw_h, tx_h, row0=row0, nrow=nrow, out_h=pinned)
    assert rel_err(out.numpy(), ref.numpy()) < 1e-6
    assert rel_err(unsplit.numpy(), ref.numpy()) < 1e-6
    pageable = torch.empty((nrow, scn.grid.nx), dtype=torch.complex64)
    out2 = plan.form_image(raw_h, tx_h, row0=row0, nrow=nrow, out_h=pageable)
    assert torch.equal(out2, ref)
    plan.close()


# ----------------------------------------------------------------------------- C5 streaming
def test_C5_streaming_frame_sampled_parity_and_chirp_shards(cuda_lib):
    """One C5 frame (chirps [f H, f H + 8192) of the long track, grid re-centred on the frame):
    sampled parity against the oracle, and the frame as the sum of 4 chirp shards (the chirp-
    sharded multi-GPU decomposition, accumulated on one GPU) equals the one-shot frame."""
    import torch

    scn = sarsim.make_config("C5")
    frames = sarsim.c5_frames(scn)
    c0, grid = frames[9]
    raw = _raw(scn)
    lo, hi = scn.antenna_box(1e-3)
    plan = cuda_lib.Plan(scn.radar, grid, scn.n_chirps, 1, (lo, hi))
    tx = torch.as_tensor(scn.tx, device="cuda:0")
    prof = plan.empty_profiles()
    plan.range_compress(raw, chirp0=c0, nchirp=8192, out=prof)
    img = plan.backproject(prof, tx, chirp0=c0, nchirp=8192)
    acc = torch.zeros_like(img)
    for k in range(4):
        plan.backproject(prof, tx, chirp0=c0 + 2048 * k, nchirp=2048, out=acc, accumulate=True)
    torch.cuda.synchronize()
    a = img.cpu().numpy()
    assert rel_err(acc.cpu().numpy(), a) < 1e-5
    sub = sarsim.Scenario("C5f", scn.radar, grid, scn.tx[c0:c0 + 8192], None, scn.targets, scn.amps,
                          np.zeros((0, 2), int), scn.wsar[c0:c0 + 8192])
    idx = sample_indices(sub, np.abs(a), stride=(97, 101), win=2)
    ref_prof = oracle_profiles(sub, raw[c0:c0 + 8192].cpu().numpy(), plan.k_lo, plan.n_bins)
    ref = oracle.backproject(ref_prof, plan.k_lo, scn.radar, sub.tx, None, grid.pixel_list(idx))
    got = a[idx[:, 0], idx[:, 1]]
    plan.close()
    assert rel_err(got, ref) <= REL_TOL
    assert np.argmax(np.abs(got)) == np.argmax(np.abs(ref))


def test_incremental_streaming_equals_one_shot_frame(cuda_lib):
    """NEXT-2: with a world-fixed grid the frame after hop h is the sum of the last 8 per-hop
    partial images; it equals one back-projection of the same 8192 chirps, and the oracle's."""
    import torch

    from paper_2306_09784_b200.stream import IncrementalStream

    scn = sarsim.make_config("C5", n_chirps=1024 * 11)
    scn.grid = sarsim.Grid(-6.0, 4.0, 0.0, 0.01, 0.01, 600, 300)
    raw = _raw(scn)
    tx = torch.as_tensor(scn.tx, device="cuda:0")
    lo, hi = scn.antenna_box(1e-3)
    st = IncrementalStream(scn.radar, scn.grid, scn.n_chirps, (lo, hi), hop=1024, hops_per_frame=8)
    for _ in range(11):
        frame = st.push(raw, tx)
    ref_plan = cuda_lib.Plan(scn.radar, scn.grid, scn.n_chirps, 1, (lo, hi))
    prof = ref_plan.range_compress(raw)
    one = ref_plan.backproject(prof, tx, chirp0=3 * 1024, nchirp=8 * 1024)
    torch.cuda.synchronize()
    f = frame.cpu().numpy()
    assert rel_err(f, one.cpu().numpy()) < 1e-5
    # the streamed frame against the oracle's BP of the frame's 8192 chirps (continuous
    # processing), on the C-6 sample of the world-fixed grid
    c0 = 3 * 1024
    sub = sarsim.Scenario("C5i-frame", scn.radar, scn.grid, scn.tx[c0:c0 + 8192], None, scn.targets, scn.amps,
                          np.zeros((0, 2), int), scn.wsar[c0:c0 + 8192])
    idx = c6_indices(sub, np.abs(f), stride=31, win=24)
    ref_prof = oracle_profiles(sub, raw[c0:c0 + 8192].cpu().numpy(), ref_plan.k_lo, ref_plan.n_bins)
    ref = oracle.backproject(ref_prof, ref_plan.k_lo, scn.radar, sub.tx, None, scn.grid.pixel_list(idx))
    got = f[idx[:, 0], idx[:, 1]]
    assert rel_err(got, ref) <= REL_TOL
    assert np.argmax(np.abs(got)) == np.argmax(np.abs(ref))
    st.close()
    ref_plan.close()


def test_image_sum_kernel(cuda_lib):
    import torch

    g = torch.Generator().manual_seed(0)
    parts = torch.randn((5, 37, 41, 2), generator=g).to("cuda:0")
    parts = torch.view_as_complex(parts.contiguous())
    out = cuda_lib.image_sum(parts)
    ref = parts[0] + parts[1] + parts[2] + parts[3] + parts[4]
    torch.cuda.synchronize()
    assert torch.allclose(out, ref, rtol=0, atol=1e-6)


# ----------------------------------------------------------------------------- full-size configs
# C-6 sample per config: (stride of whole rows / columns, window half-width); C4 (36 Mpx x 4 RX) is
# thinned to keep its oracle leg near a minute on 16 host cores
C6_PROTOCOL = {"C2": (31, 24), "C3": (31, 24), "C0": (31, 24), "C6": (31, 24), "C4": (191, 12)}


@pytest.mark.parametrize("cfg", ["C2", "C3", "C0", "C4", "C6"])
def test_full_size_config_sampled_parity(cuda_lib, cfg):
    """BASELINE configs at full size in the bench's launch configuration, against the oracle on
    the C-6 protocol sample: whole rows and columns at a stride coprime with the 32-px tile (every
    tile offset, the ragged last tile row and column included), +-24 px windows around every
    isolated target and the GPU's 32 largest pixels (C3: ~0.85 M px x 8192 chirps)."""
    scn = sarsim.make_config(cfg)
    raw = _raw(scn)
    img, prof, plan = gpu_image(scn, raw, return_prof=True)
    a = np.abs(img.cpu().numpy())
    g = scn.grid
    stride, win = C6_PROTOCOL[cfg]
    idx = c6_indices(scn, a, stride=stride, win=win)
    assert np.any(idx[:, 0] == g.ny - 1) and np.any(idx[:, 1] == g.nx - 1)
    pix = g.pixel_list(idx)
    # oracle on the crop the plan keeps (it raises if any pixel needed a bin outside it)
    ref_prof = oracle_profiles(scn, raw.cpu().numpy(), plan.k_lo, plan.n_bins)
    ref = oracle.backproject(ref_prof, plan.k_lo, scn.radar, scn.tx, scn.rx, pix)
    got = img.cpu().numpy()[idx[:, 0], idx[:, 1]]
    plan.close()
    assert rel_err(got, ref) <= REL_TOL
    # global peak: the oracle's maximum over the sample (which holds windows around the GPU's
    # maxima) sits at the GPU's global argmax; with the 7 m apertures that is the pole (a = 1)
    k = np.argmax(np.abs(ref))
    assert tuple(idx[k]) == np.unravel_index(np.argmax(a), a.shape)
    if cfg != "C6":    # C6's 8 cm aperture resolves ~0.2 m in azimuth: the wall outshines the pole
        assert tuple(idx[k]) == tuple(scn.isolated[0])
    # local argmax of every isolated target agrees (within its sampled window) wherever the
    # oracle's peak is unambiguous (best/second > 1 + 4e-3, reading A15)
    for (j, i) in scn.isolated:
        sel = (np.abs(idx[:, 0] - j) <= 2) & (np.abs(idx[:, 1] - i) <= 2)
        r = np.sort(np.abs(ref[sel]))
        if r[-1] > (1 + 4e-3) * r[-2]:
            assert np.argmax(np.abs(got[sel])) == np.argmax(np.abs(ref[sel]))


def test_zero_input_gives_zero_image(cuda_lib):
    """T9 on the GPU: zero raw samples give exactly zero profiles and a zero image (monostatic and
    bistatic, unsplit and chirp-split launches)."""
    import torch

    for n_rx, nchirp in ((1, 100), (3, 2048)):
        scn = sarsim.small_config(n_chirps=nchirp, ns=128, nx=40, ny=33, seed=61, n_rx=n_rx)
        raw = torch.zeros((nchirp, n_rx, 128), dtype=torch.float32, device="cuda:0")
        img, prof, plan = gpu_image(scn, raw, return_prof=True)
        torch.cuda.synchronize()
        assert torch.count_nonzero(prof) == 0 and torch.count_nonzero(img) == 0
        plan.close()


@pytest.mark.parametrize("shape", ["4,4", "4,8", "8,8", "8,4,2,8", "8,4,5,4"])
@pytest.mark.parametrize("n_rx", [1, 3])
def test_cta_shapes_and_rings_match_oracle(cuda_lib, shape, n_rx, monkeypatch):
    """Every supported CTA shape / ring configuration (SAR_BP_SHAPE="ncw,pb[,stages,cb]", the
    tuning override; 4,4 is also the default of wide-window polar plans) meets the parity bar."""
    monkeypatch.setenv("SAR_BP_SHAPE", shape)
    scn = sarsim.small_config(n_chirps=72, ns=256, nx=70, ny=45, n_rx=n_rx, curved=n_rx > 1, seed=61)
    raw = _raw(scn)
    got = gpu_image(scn, raw).cpu().numpy().reshape(-1)
    ref = oracle_image(scn, raw.cpu().numpy())
    assert np.argmax(np.abs(got)) == np.argmax(np.abs(ref))
    assert rel_err(got, ref) <= REL_TOL


def test_producer_built_windows_match_pair_rows(cuda_lib, monkeypatch):
    """The BP producer's own window construction (used when the pair-format rows cannot be
    allocated; forced here with SAR_BP_NO_PAIRS=1 in a fresh process) gives the same image."""
    import os
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, %r); import numpy as np, torch, sarsim\n"
            "from tests.helpers import gpu_image\n"
            "scn = sarsim.small_config(n_chirps=80, ns=256, nx=70, ny=45, n_rx=2, curved=True, seed=62)\n"
            "raw = sarsim.simulate_raw(scn, device='cuda:0')\n"
            "np.save(sys.argv[1], gpu_image(scn, raw).cpu().numpy())\n") % os.getcwd()
    outs = []
    for flag in ("0", "1"):
        path = f"/tmp/_sar_np_{os.getpid()}_{flag}.npy"
        env = dict(os.environ, SAR_BP_NO_PAIRS=flag)
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env)
        outs.append(np.load(path))
    # same per-entry arithmetic in both places; allow FMA-contraction differences
    assert np.abs(outs[0] - outs[1]).max() <= 1e-6 * np.abs(outs[0]).max()


@pytest.mark.parametrize("shape", [None, "8,4,3,4"])
def test_sixteen_rx_array_matches_oracle(cuda_lib, shape, monkeypatch):
    """The paper's reference setup: 16 RX (Table 1; Measure F keeps 8).  With the override 4
    chirps x 16 RX = 64 items share a ring stage (more items than producer lanes)."""
    if shape:
        monkeypatch.setenv("SAR_BP_SHAPE", shape)
    scn = sarsim.small_config(n_chirps=40, ns=256, nx=45, ny=36, n_rx=16, seed=63)
    raw = _raw(scn)
    got = gpu_image(scn, raw).cpu().numpy().reshape(-1)
    ref = oracle_image(scn, raw.cpu().numpy())
    assert np.argmax(np.abs(got)) == np.argmax(np.abs(ref))
    assert rel_err(got, ref) <= REL_TOL


def test_largest_fft_and_full_crop_match_oracle(cuda_lib):
    """Maximum transform size (fft_len = 16384, Ns = 2048: 128 KB of shared memory per FFT) and
    the smallest range-bin spacing (Z = 8 over 2048 samples)."""
    scn = sarsim.small_config(n_chirps=24, ns=2048, nx=40, ny=30, seed=64)
    assert scn.radar.fft_len == 16384
    raw = _raw(scn)
    img, prof, plan = gpu_image(scn, raw, return_prof=True)
    ref_prof = oracle_profiles(scn, raw.cpu().numpy(), plan.k_lo, plan.n_bins)
    got_prof = prof.cpu().numpy()
    assert np.abs(got_prof - ref_prof).max() <= 1e-5 * np.abs(ref_prof).max()
    got = img.cpu().numpy().reshape(-1)
    ref = oracle_image(scn, raw.cpu().numpy())
    plan.close()
    assert np.argmax(np.abs(got)) == np.argmax(np.abs(ref))
    assert rel_err(got, ref) <= REL_TOL


def test_bounds_check_build_counts_no_violation():
    """The -DSAR_DEBUG_CHECKS build of the same sources (compute-sanitizer is closed on this GPU
    pool) over every kernel family: no window index outside its item, no workspace plane out of
    range, no clamped bulk copy for inputs within the contract, and no shared-memory read outside
    the allocation even for an antenna outside the declared box (tools/check_cases.py)."""
    import os
    import subprocess
    import sys

    from paper_2306_09784_b200 import _build

    if not os.path.exists(_build.CHECK_LIB):
        _build.build(out=_build.CHECK_LIB, defines=["-DSAR_DEBUG_CHECKS"])
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "check_cases.py")], capture_output=True,
                         text=True, timeout=600, env={**os.environ, "SAR_LIB": _build.CHECK_LIB}, cwd=root)
    assert out.returncode == 0, out.stdout + out.stderr[-3000:]
    assert out.stdout.count("-> ok") >= 10
