"""Ad-hoc GPU probe: MUFU sin/cos accuracy vs argument size, and BP/RC timings on C0/C2/C3."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("SAR_PKG_ROOT"):   # tuning: another build's package (e.g. a previous commit)
    sys.path.insert(0, os.environ["SAR_PKG_ROOT"])
import numpy as np
import torch
import sarsim
from paper_2306_09784_b200 import sar

dev = torch.device("cuda:0")
print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0).multi_processor_count)

def time_cfg(name, reps=5):
    scn = sarsim.make_config(name)
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    lo, hi = scn.antenna_box(1e-3)
    plan = sar.Plan(scn.radar, scn.grid, scn.n_chirps, scn.n_rx, (lo, hi))
    tx = torch.as_tensor(scn.tx, device=dev)
    rx = None if scn.rx is None else torch.as_tensor(scn.rx, device=dev).contiguous()
    prof = plan.range_compress(raw)
    img = plan.backproject(prof, tx, rx)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    trc, tbp = [], []
    for _ in range(reps):
        e[0].record(); plan.range_compress(raw, out=prof); e[1].record(); plan.backproject(prof, tx, rx, out=img); e[2].record()
        torch.cuda.synchronize()
        trc.append(e[0].elapsed_time(e[1])); tbp.append(e[1].elapsed_time(e[2]))
    upd = scn.updates
    print(f"{name}: info {plan.info.as_dict()}")
    print(f"{name}: rc {min(trc):.3f} ms  bp {min(tbp):.3f} ms  -> {upd/min(tbp)/1e-3:.3e} upd/s")
    plan.close()

for n in sys.argv[1:] or ["C0", "C2", "C3"]:
    time_cfg(n)
