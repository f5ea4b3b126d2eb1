"""Per-rank work of the N-GPU pixel-row bench on one GPU: sar_backproject of the rank's rows
(chirp split) vs sar_backproject_scatter of the same rows into N local full images standing in
for the peers (split scatter: the last chunk of each tile publishes).  No cross-rank waits."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import sarsim
from paper_2306_09784_b200 import sar
from paper_2306_09784_b200.dist import row_partition

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
dev = torch.device("cuda:0")
scn = sarsim.make_config(cfg)
raw = sarsim.simulate_raw(scn, device="cuda:0")
lo, hi = scn.antenna_box(1e-3)
g = scn.grid
plan = sar.Plan(scn.radar, g, scn.n_chirps, scn.n_rx, (lo, hi))
tx = torch.as_tensor(scn.tx, device=dev)
prof = plan.range_compress(raw)
for world in (2, 4, 8):
    row0, nrow = row_partition(g.ny, world, 0)
    imgs = [torch.zeros((g.ny, g.nx), dtype=torch.complex64, device=dev) for _ in range(world)]
    out = torch.empty((nrow, g.nx), dtype=torch.complex64, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for it in range(3):
        ev[0].record()
        plan.backproject(prof, tx, row0=row0, nrow=nrow, out=out)
        ev[1].record()
        plan.backproject_scatter(prof, tx, [im.data_ptr() for im in imgs], row0=row0, nrow=nrow)
        ev[2].record()
        torch.cuda.synchronize()
    err = float((imgs[-1][row0:row0 + nrow] - out).abs().max() / out.abs().max())
    print(f"{cfg} N={world}: rows {nrow}: backproject {ev[0].elapsed_time(ev[1]):.3f} ms, "
          f"scatter to {world} images {ev[1].elapsed_time(ev[2]):.3f} ms, rel diff {err:.1e}")
plan.close()
