"""Per-rank work of the N-GPU bench legs on one GPU (no cross-rank waits), every rank of N = 2/4/8:
  fused leg -- sar_backproject_scatter_tiles of the rank's tile block into N local full images
              standing in for the peers (unsplit, or split with the last chunk publishing);
  NCCL leg  -- sar_backproject of the rank's whole tile rows (the all-gather itself not included).
Prints per-rank ms and the max over ranks against the 1-GPU image time / N (the ideal)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import sarsim
from paper_2306_09784_b200 import sar
from paper_2306_09784_b200.dist import rebalance, row_partition, tile_partition

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
worlds = [int(w) for w in sys.argv[2:]] or [2, 4, 8]
dev = torch.device("cuda:0")
scn = sarsim.make_config(cfg)
raw = sarsim.simulate_raw(scn, device="cuda:0")
lo, hi = scn.antenna_box(1e-3)
g = scn.grid
plan = sar.Plan(scn.radar, g, scn.n_chirps, scn.n_rx, (lo, hi))
tx = torch.as_tensor(scn.tx, device=dev)
rx = None if scn.rx is None else torch.as_tensor(scn.rx, device=dev).contiguous()
prof = plan.range_compress(raw)
tiles_x, tiles_y = plan.tiles
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, reps=2):
    best = 1e30
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


full = plan.empty_image()
t1 = timed(lambda: plan.backproject(prof, tx, rx, out=full))
print(f"{cfg} 1-GPU backproject {t1:.3f} ms")
for world in worlds:
    imgs = [torch.zeros((g.ny, g.nx), dtype=torch.complex64, device=dev) for _ in range(min(world, 8))]
    ptrs = [im.data_ptr() for im in imgs]
    ideal = t1 / world
    # bench.py's measured load balance: equal blocks, then two re-cuts on the measured block times
    tb = [tile_partition(tiles_x * tiles_y, world, r) for r in range(world)]
    pb = list(tb)
    rb = [row_partition(tiles_y, world, r) for r in range(world)]
    ty = plan.info.tile_y
    for it in range(3):
        fused = [timed(lambda: plan.backproject_scatter_tiles(prof, tx, ptrs, t0, nt, rx)) for t0, nt in tb]
        pub = [timed(lambda: plan.backproject_scatter_tiles(prof, tx, ptrs, t0, nt, rx, publish=True)) for t0, nt in pb]
        if os.environ.get("PROBE_PLAIN_TILES"):   # the same tile blocks through the plain family
            plain = [timed(lambda: plan.backproject_tiles(prof, tx, t0, nt, rx, out=imgs[0])) for t0, nt in tb]
            print(f"N={world} it{it}: plain tile blocks per rank {['%.3f' % t for t in plain]} max {max(plain):.3f} "
                  f"({max(plain) / ideal:.3f} x ideal)")
        rows = []
        for a, n in rb:
            row0, nrow = min(g.ny, a * ty), min(g.ny, (a + n) * ty) - min(g.ny, a * ty)
            out = torch.empty((max(nrow, 1), g.nx), dtype=torch.complex64, device=dev)
            rows.append(timed(lambda: plan.backproject(prof, tx, rx, row0=row0, nrow=nrow, out=out[:nrow])))
        label = "equal blocks" if it == 0 else f"rebalanced x{it}"
        for name, ts in (("fused (tile blocks)", fused), ("publish (tile blocks)", pub), ("NCCL leg (tile rows)", rows)):
            print(f"N={world} {label}: {name} per rank {['%.3f' % t for t in ts]} max {max(ts):.3f} "
                  f"({max(ts) / ideal:.3f} x ideal, spread {(max(ts) - min(ts)) / max(ts):.1%})")
        tb = [rebalance(tb, fused, world, r) for r in range(world)]
        pb = [rebalance(pb, pub, world, r) for r in range(world)]
        rb = [rebalance(rb, rows, world, r) for r in range(world)]
    del imgs
plan.close()
