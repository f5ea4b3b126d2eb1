"""One warm-up + profiled back-projections of a row shard of a config (for ncu of a rank's kernel).

usage: prof_shard.py CFG ROW0 NROW [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("SAR_PKG_ROOT"):   # tuning: another build's package (e.g. a previous commit)
    sys.path.insert(0, os.environ["SAR_PKG_ROOT"])
import torch

import sarsim
from paper_2306_09784_b200 import sar

cfg = sys.argv[1]
row0, nrow = int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
scn = sarsim.make_config(cfg)
dev = torch.device("cuda:0")
raw = sarsim.simulate_raw(scn, device="cuda:0")
lo, hi = scn.antenna_box(1e-3)
plan = sar.Plan(scn.radar, scn.grid, scn.n_chirps, scn.n_rx, (lo, hi))
tx = torch.as_tensor(scn.tx, device=dev)
rx = None if scn.rx is None else torch.as_tensor(scn.rx, device=dev).contiguous()
prof = plan.range_compress(raw)
out = torch.empty((nrow, scn.grid.nx), dtype=torch.complex64, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(reps):
    e0.record()
    plan.backproject(prof, tx, rx, row0=row0, nrow=nrow, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(cfg, row0, nrow, "bp ms %.3f" % e0.elapsed_time(e1), flush=True)
