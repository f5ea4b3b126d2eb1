import os, sys
sys.path.insert(0, "/root/repo")
import torch, sarsim
from paper_2306_09784_b200 import sar
from paper_2306_09784_b200.dist import row_partition
scn = sarsim.make_config("C3"); dev = torch.device("cuda:0")
raw = sarsim.simulate_raw(scn, device="cuda:0"); lo, hi = scn.antenna_box(1e-3); g = scn.grid
plan = sar.Plan(scn.radar, g, scn.n_chirps, scn.n_rx, (lo, hi))
tx = torch.as_tensor(scn.tx, device=dev); prof = plan.range_compress(raw)
print("tile_y", plan.info.tile_y)
for world in (8,):
    ts = []
    for r in range(world):
        row0, nrow = row_partition(g.ny, world, r)
        out = torch.empty((nrow, g.nx), dtype=torch.complex64, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for it in range(2):
            e0.record(); plan.backproject(prof, tx, row0=row0, nrow=nrow, out=out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(world, ["%.3f" % t for t in ts])
# aligned partitions: multiples of 32 rows
for rows in [(0, 352), (352, 384), (0, 384)]:
    out = torch.empty((rows[1], g.nx), dtype=torch.complex64, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(2):
        e0.record(); plan.backproject(prof, tx, row0=rows[0], nrow=rows[1], out=out); e1.record(); torch.cuda.synchronize()
    print(rows, "%.3f" % e0.elapsed_time(e1))
