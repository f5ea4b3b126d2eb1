"""sar_form_image (host buffers) vs the device-resident step for one config: event times and
the kernel list (run under ncu --metrics gpu__time_duration.sum for per-kernel times)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import sarsim
from paper_2306_09784_b200 import sar

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
dev = torch.device("cuda:0")
scn = sarsim.make_config(cfg)
raw = sarsim.simulate_raw(scn, device="cuda:0")
lo, hi = scn.antenna_box(1e-3)
g = scn.grid
plan = sar.Plan(scn.radar, g, scn.n_chirps, scn.n_rx, (lo, hi))
tx = torch.as_tensor(scn.tx, device=dev)
raw_h = raw.cpu().pin_memory()
tx_h = torch.as_tensor(scn.tx).contiguous().pin_memory()
img_h = torch.empty((g.ny, g.nx), dtype=torch.complex64).pin_memory()
prof = plan.empty_profiles()
img = plan.empty_image()
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for it in range(3):
    e[0].record()
    plan.range_compress(raw, out=prof)
    plan.backproject(prof, tx, out=img)
    e[1].record()
    plan.form_image(raw_h, tx_h, out_h=img_h, sync=False)
    e[2].record()
    torch.cuda.synchronize()
print(f"{cfg}: device step {e[0].elapsed_time(e[1]):.3f} ms, form_image {e[1].elapsed_time(e[2]):.3f} ms")
plan.close()
