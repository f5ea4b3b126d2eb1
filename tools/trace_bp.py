"""Ring-wait trace of bp_kernel (tuning build with -DSAR_BP_TRACE, via SAR_LIB): per traced CTA,
consumer warps' full-barrier waits and per-stage work, the producer's empty waits and fill times,
and each warp's hardware warp slot (SMSP = warpid % 4)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import sarsim
from paper_2306_09784_b200 import sar

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
scn = sarsim.make_config(cfg)
dev = torch.device("cuda:0")
raw = sarsim.simulate_raw(scn, device="cuda:0")
lo, hi = scn.antenna_box(1e-3)
plan = sar.Plan(scn.radar, scn.grid, scn.n_chirps, scn.n_rx, (lo, hi))
tx = torch.as_tensor(scn.tx, device=dev)
prof = plan.range_compress(raw)
img = plan.backproject(prof, tx)
torch.cuda.synchronize()
img = plan.backproject(prof, tx, out=img)
torch.cuda.synchronize()
tr = np.zeros((4, 9, 256, 3), np.uint64)
wid = np.zeros((4, 9, 2), np.uint32)
lib = sar.load()
lib.sar_debug_trace(tr.ctypes.data_as(ctypes.c_void_p), wid.ctypes.data_as(ctypes.c_void_p))
S = plan.info.chirps_per_stage
for c in range(4):
    t = tr[c].astype(np.int64)
    n = 200
    print(f"CTA {c}: smid {wid[c, 0, 1]} warpids {list(wid[c, :, 0])}")
    wait = (t[:8, 1:n, 1] - t[:8, 1:n, 0])
    work = (t[:8, 1:n, 2] - t[:8, 1:n, 1])
    tot = (t[:8, n, 0] - t[:8, 1, 0])
    for w in range(8):
        print(f"  consumer warp {w} (smsp {wid[c, w, 0] % 4}): wait {wait[w].sum() / tot[w]:.3f} of time, "
              f"work/stage {np.median(work[w]):.0f} clk, lag vs warp0 at stage {n}: {t[w, n, 0] - t[0, n, 0]} clk")
    pw = t[8, 1:n, 1] - t[8, 1:n, 0]
    pf = t[8, 1:n, 2] - t[8, 1:n, 1]
    print(f"  producer (smsp {wid[c, 8, 0] % 4}): empty-wait {pw.sum() / (t[8, n, 0] - t[8, 1, 0]):.3f}, "
          f"fill median {np.median(pf):.0f} clk, p90 {np.percentile(pf, 90):.0f}")
    # how far ahead is the producer when consumers wait: fill completion vs consumer wait end
    ready = t[8, :n, 2]
    late = [(t[:8, k, 1].max() - ready[k]) for k in range(1, n)]
    print(f"  stage ready -> last consumer start: median {np.median(late):.0f} clk")
