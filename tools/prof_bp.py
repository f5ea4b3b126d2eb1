"""One warm-up + one profiled range compression + back-projection of a config (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import sarsim
from paper_2306_09784_b200 import sar

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
scn = sarsim.make_config(cfg)
dev = torch.device("cuda:0")
raw = sarsim.simulate_raw(scn, device="cuda:0")
lo, hi = scn.antenna_box(1e-3)
plan = sar.Plan(scn.radar, scn.grid, scn.n_chirps, scn.n_rx, (lo, hi))
tx = torch.as_tensor(scn.tx, device=dev)
rx = None if scn.rx is None else torch.as_tensor(scn.rx, device=dev).contiguous()
prof = plan.empty_profiles()
img = plan.empty_image()
for _ in range(reps):
    plan.range_compress(raw, out=prof)
    plan.backproject(prof, tx, rx, out=img)
torch.cuda.synchronize()
print(cfg, "ok", float(img.abs().max()))
