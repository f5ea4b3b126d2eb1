"""N > 1 path on CPU (-m "not gpu"): world_size-2 gloo process groups exercise the row and
chirp partitioning and the collectives of paper_2306_09784_b200.dist.  The per-rank compute
is the oracle (a CPU stand-in for the CUDA kernels); the result must equal the unsharded
oracle image."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import sarsim
from paper_2306_09784_b200.dist import (chirp_partition, gather_rows, rebalance, reduce_partials, row_partition,
                                       tile_partition, tile_row_partition, weighted_partition)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    scn = sarsim.small_config(n_chirps=24, ns=64, nx=14, ny=11, seed=3, n_rx=2)
    raw = sarsim.simulate_raw(scn).numpy()
    prof = oracle.range_compress(raw, scn.radar.fft_len, 1, scn.wsar)
    return scn, prof


def _worker(rank, world, port, mode, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scn, prof = _scene()
        g = scn.grid
        if mode in ("rows", "tile_rows"):
            if mode == "rows":
                parts = None
                r0, n = row_partition(g.ny, world, rank)
            else:   # whole tile rows of 4 px: 11 rows = 3 tile rows -> ragged blocks 8 + 3
                parts = [tile_row_partition(-(-g.ny // 4), 4, g.ny, world, r) for r in range(world)]
                r0, n = parts[rank]
            pix = g.pixels(rows=np.arange(r0, r0 + n))
            loc = oracle.backproject(prof, 0, scn.radar, scn.tx, scn.rx, pix, nthreads=1)
            local = torch.from_numpy(loc.astype(np.complex64).reshape(n, g.nx))
            full = gather_rows(local, g.ny, parts=parts)
            if rank == 0:
                out_q.put(full.numpy())
        else:
            c0, nc = chirp_partition(scn.n_chirps, world, rank)
            sl = slice(c0, c0 + nc)
            part = oracle.backproject(prof[sl], 0, scn.radar, scn.tx[sl], scn.rx[sl], g.pixels(), nthreads=1)
            t = torch.from_numpy(part.astype(np.complex64).reshape(g.ny, g.nx)).contiguous()
            reduce_partials(t, dst=0)
            if rank == 0:
                out_q.put(t.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["rows", "tile_rows", "chirps"])
def test_two_rank_gloo_sharding_equals_unsharded(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    scn, prof = _scene()
    ref = oracle.backproject(prof, 0, scn.radar, scn.tx, scn.rx, scn.grid.pixels()).reshape(got.shape)
    assert np.abs(got - ref).max() <= 1e-6 * np.abs(ref).max()


def test_partitions_cover_exactly():
    for n in (1, 7, 3000, 1201):
        for w in (1, 2, 3, 4, 8):
            blocks = [row_partition(n, w, r) for r in range(w)]
            assert blocks[0][0] == 0
            for (a, na), (b, _) in zip(blocks, blocks[1:]):
                assert a + na == b
            assert sum(nb for _, nb in blocks) == n
            assert max(nb for _, nb in blocks) - min(nb for _, nb in blocks) <= 1


def test_tile_partitions_cover_exactly():
    """Tile blocks are balanced to +-1 tile; tile-row blocks are whole tile rows (+-1 tile row)
    covering the grid rows exactly (C3: 94 tile rows of 32 px, ragged last row)."""
    for nt in (1, 9, 8836, 94 * 38):
        for w in (1, 2, 3, 8):
            blocks = [tile_partition(nt, w, r) for r in range(w)]
            assert sum(b for _, b in blocks) == nt and blocks[0][0] == 0
            assert max(b for _, b in blocks) - min(b for _, b in blocks) <= 1
    for ny, ty in ((3000, 32), (1201, 32), (90, 16), (7, 32)):
        tiles_y = -(-ny // ty)
        for w in (1, 2, 4, 8):
            parts = [tile_row_partition(tiles_y, ty, ny, w, r) for r in range(w)]
            assert parts[0][0] == 0 and sum(n for _, n in parts) == ny
            for (a, na), (b, _) in zip(parts, parts[1:]):
                assert a + na == b and (na == 0 or a % ty == 0)
            full = [n for _, n in parts if n > 0][:-1]
            assert all(n % ty == 0 for n in full)


def test_weighted_partition_and_measured_rebalance():
    """Cost-balanced contiguous blocks (bench.py's measured load balance): they cover the items
    exactly, equal weights give blocks balanced to +-1 item, and re-cutting equal blocks on measured
    block times whose cost per item falls with the index (C3: tile rows near the track cost more)
    brings the predicted per-rank costs within one item's cost of each other."""
    for n in (8, 94, 8836):
        for w in (1, 2, 3, 8):
            blocks = [weighted_partition([1.0] * n, w, r) for r in range(w)]
            assert blocks[0][0] == 0 and sum(b for _, b in blocks) == n
            for (a, na), (b, _) in zip(blocks, blocks[1:]):
                assert a + na == b
            assert max(b for _, b in blocks) - min(b for _, b in blocks) <= 1
    cost = [1.0 + 0.1 * (1.0 - i / 8835) for i in range(8836)]   # true per-tile cost
    for w in (2, 4, 8):
        blocks = [tile_partition(8836, w, r) for r in range(w)]
        for _ in range(3):
            times = [sum(cost[a:a + n]) for a, n in blocks]
            blocks = [rebalance(blocks, times, w, r) for r in range(w)]
            assert blocks[0][0] == 0 and sum(n for _, n in blocks) == 8836
        times = [sum(cost[a:a + n]) for a, n in blocks]
        assert max(times) - min(times) <= 2 * max(cost)
    assert weighted_partition([0.0] * 5, 2, 0) == row_partition(5, 2, 0)   # no measured cost: equal blocks
