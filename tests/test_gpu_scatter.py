"""NEXT-4 fused gather on one GPU: the BP scatter epilogue (sar_backproject_scatter) writes the
rank's rows into several full images at once -- here local buffers standing in for P2P-mapped
peers (no cross-rank waiting is involved), and, where the NVSwitch supports it, a one-rank
symmetric-memory multicast address (multimem.st).  Rows outside the shard stay untouched and
the stored rows equal sar_backproject's bit for bit."""
import numpy as np
import pytest

import sarsim

pytestmark = pytest.mark.gpu


def _setup(cuda_lib):
    import torch

    scn = sarsim.small_config(n_chirps=64, ns=256, nx=77, ny=70, seed=51)
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    lo, hi = scn.antenna_box(1e-3)
    plan = cuda_lib.Plan(scn.radar, scn.grid, scn.n_chirps, 1, (lo, hi))
    tx = torch.as_tensor(scn.tx, device="cuda:0")
    prof = plan.range_compress(raw)
    return scn, plan, tx, prof


@pytest.mark.parametrize("rows", [(0, 70), (32, 32), (13, 40)])
def test_scatter_to_several_images_equals_backproject(cuda_lib, rows):
    import torch

    scn, plan, tx, prof = _setup(cuda_lib)
    row0, nrow = rows
    g = scn.grid
    ref = plan.backproject(prof, tx, row0=row0, nrow=nrow)
    imgs = [torch.full((g.ny, g.nx), complex(7.0, -7.0), dtype=torch.complex64, device="cuda:0") for _ in range(3)]
    plan.backproject_scatter(prof, tx, [im.data_ptr() for im in imgs], row0=row0, nrow=nrow)
    torch.cuda.synchronize()
    for im in imgs:
        assert torch.equal(im[row0:row0 + nrow], ref)
        assert torch.all(im[:row0] == complex(7.0, -7.0)) and torch.all(im[row0 + nrow:] == complex(7.0, -7.0))
    plan.close()


def test_scatter_argument_errors(cuda_lib):
    from paper_2306_09784_b200 import sar

    scn, plan, tx, prof = _setup(cuda_lib)
    with pytest.raises(sar.SarError):
        plan.backproject_scatter(prof, tx, [])
    with pytest.raises(sar.SarError):
        plan.backproject_scatter(prof, tx, [prof.data_ptr()] * 9)
    with pytest.raises(sar.SarError):
        plan.backproject_scatter(prof, tx, [prof.data_ptr(), prof.data_ptr()], multicast=True)
    plan.close()


def test_symmetric_memory_one_rank(cuda_lib):
    """The bench's N > 1 path on a one-rank group: symmetric-memory image, scatter epilogue
    through the multicast address when available (else the rank's own mapped buffer)."""
    import torch
    import torch.distributed as dist

    from paper_2306_09784_b200.dist import FusedRowGather

    scn, plan, tx, prof = _setup(cuda_lib)
    g = scn.grid
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1,
                                device_id=torch.device("cuda:0"))
    try:
        fg = FusedRowGather(g.ny, g.nx, torch.device("cuda:0"))
        fg.image.fill_(complex(3.0, 3.0))
        torch.cuda.synchronize()
        plan.backproject_scatter(prof, tx, fg.ptrs, multicast=fg.multicast)
        fg.barrier()
        torch.cuda.synchronize()
        ref = plan.backproject(prof, tx)
        torch.cuda.synchronize()
        assert torch.equal(fg.image, ref), f"multicast={fg.multicast}"
        print("multicast path:", fg.multicast)
    finally:
        plan.close()
        if own:
            dist.destroy_process_group()


def test_scatter_add_chirp_shards_equal_full_image(cuda_lib):
    """The fused chirp-shard reduction: shards added by the epilogue into zeroed images (two
    destinations) equal the one-launch image to fp32 summation order (with one rsqrt leg per
    chirp; the shards regroup derived legs otherwise: 1e-4, reading A22)."""
    import torch

    import os

    scn, plan, tx, prof = _setup(cuda_lib)
    g = scn.grid
    for derive, tol in (("1", 1e-4), ("0", 1e-5)):
        os.environ["SAR_BP_DERIVE"] = derive
        try:
            ref = plan.backproject(prof, tx)
            imgs = [torch.zeros((g.ny, g.nx), dtype=torch.complex64, device="cuda:0") for _ in range(2)]
            for c0, nc in [(0, 20), (20, 30), (50, 14)]:
                plan.backproject_scatter(prof, tx, [im.data_ptr() for im in imgs], chirp0=c0, nchirp=nc, add=True)
            torch.cuda.synchronize()
        finally:
            del os.environ["SAR_BP_DERIVE"]
        for im in imgs:
            err = float((im - ref).abs().max() / ref.abs().max())
            assert err < tol, (derive, err)
    plan.close()


@pytest.mark.parametrize("rows,n_rx", [((0, 24), 1), ((5, 13), 1), ((3, 17), 3)])
def test_chirp_split_scatter_last_chunk_publishes(cuda_lib, rows, n_rx):
    """A scatter whose grid is too small to fill the GPU runs chirp-split: every chunk stores its
    partial tile into its own workspace plane and the last chunk of each tile (per-tile counter)
    sums the planes in chunk order and stores the finished tile to every destination.  Equals
    sar_backproject (same chunks, same order) bit for bit, the oracle to the parity bar; rows
    outside the shard untouched."""
    import torch

    from tests.helpers import REL_TOL, oracle_image, rel_err

    scn = sarsim.small_config(n_chirps=4096 // n_rx, ns=128, nx=40, ny=24, seed=57, n_rx=n_rx)
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    lo, hi = scn.antenna_box(1e-3)
    plan = cuda_lib.Plan(scn.radar, scn.grid, scn.n_chirps, n_rx, (lo, hi))
    rx = None if n_rx == 1 else torch.as_tensor(scn.rx, device="cuda:0").contiguous()
    # 2 tiles of 32 x 32 px and 4096 chirps: the launcher splits into 8 chunks of 512 chirps
    tx = torch.as_tensor(scn.tx, device="cuda:0")
    prof = plan.range_compress(raw)
    row0, nrow = rows
    g = scn.grid
    ref = plan.backproject(prof, tx, rx, row0=row0, nrow=nrow)
    imgs = [torch.full((g.ny, g.nx), complex(7.0, -7.0), dtype=torch.complex64, device="cuda:0") for _ in range(3)]
    for _ in range(2):   # the workspace (counters, chunk planes) is reset per launch
        plan.backproject_scatter(prof, tx, [im.data_ptr() for im in imgs], rx, row0=row0, nrow=nrow)
    torch.cuda.synchronize()
    ora = oracle_image(scn, raw.cpu().numpy()).reshape(g.ny, g.nx)[row0:row0 + nrow]
    for im in imgs:
        got = im[row0:row0 + nrow].cpu().numpy()
        assert torch.equal(im[row0:row0 + nrow], ref)
        assert rel_err(got, ora) <= REL_TOL
        assert torch.all(im[:row0] == complex(7.0, -7.0)) and torch.all(im[row0 + nrow:] == complex(7.0, -7.0))
    plan.close()


def test_tile_scatter_equals_tile_backproject(cuda_lib):
    """sar_backproject_scatter_tiles: a rank's block of absolute tiles stored into every full
    image; equals sar_backproject_tiles bit for bit, other pixels untouched."""
    import torch

    scn, plan, tx, prof = _setup(cuda_lib)
    g = scn.grid
    tiles_x, tiles_y = plan.tiles
    sentinel = complex(7.0, -7.0)
    ref = torch.full((g.ny, g.nx), sentinel, dtype=torch.complex64, device="cuda:0")
    plan.backproject_tiles(prof, tx, 2, 3, out=ref)
    imgs = [torch.full((g.ny, g.nx), sentinel, dtype=torch.complex64, device="cuda:0") for _ in range(2)]
    plan.backproject_scatter_tiles(prof, tx, [im.data_ptr() for im in imgs], 2, 3)
    torch.cuda.synchronize()
    assert int((ref != sentinel).sum()) > 0
    for im in imgs:
        assert torch.equal(im, ref)
    plan.close()


@pytest.mark.parametrize("big", [False, True])
def test_publish_scatter_equals_tile_backproject(cuda_lib, big):
    """SAR_SCATTER_PUBLISH: the tiles are computed into images[0] like sar_backproject_tiles (bit for
    bit), then copied to images[1..]; other pixels untouched.  ``big``: a C3 tile block whose launch
    splits its chirps (chunk planes + split sum before the copy), ragged last tile row included."""
    import torch

    from paper_2306_09784_b200 import sar

    if big:
        scn = sarsim.make_config("C3")
        raw = sarsim.simulate_raw(scn, device="cuda:0")
        lo, hi = scn.antenna_box(1e-3)
        plan = sar.Plan(scn.radar, scn.grid, scn.n_chirps, scn.n_rx, (lo, hi))
        tx = torch.as_tensor(scn.tx, device="cuda:0")
        prof = plan.range_compress(raw)
        tiles_x, tiles_y = plan.tiles
        t0, nt = tiles_x * tiles_y - 1111, 1111   # the last 1111 tiles: ragged last row and column
    else:
        scn, plan, tx, prof = _setup(cuda_lib)
        t0, nt = 2, 3
    g = scn.grid
    sentinel = complex(7.0, -7.0)
    ref = torch.full((g.ny, g.nx), sentinel, dtype=torch.complex64, device="cuda:0")
    plan.backproject_tiles(prof, tx, t0, nt, out=ref)
    imgs = [torch.full((g.ny, g.nx), sentinel, dtype=torch.complex64, device="cuda:0") for _ in range(3)]
    plan.backproject_scatter_tiles(prof, tx, [im.data_ptr() for im in imgs], t0, nt, publish=True)
    torch.cuda.synchronize()
    assert int((ref != sentinel).sum()) > 0
    for im in imgs:
        assert torch.equal(im, ref)
    with pytest.raises(sar.SarError):
        plan.backproject_scatter_tiles(prof, tx, [imgs[0].data_ptr()], t0, nt, publish=True, add=True)
    plan.close()
