"""Where does the GPU-vs-oracle error come from?  rc vs bp, and its spatial pattern."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, sarsim
from paper_2306_09784_b200 import sar

def run(scn, tag):
    dev = torch.device("cuda:0")
    raw = sarsim.simulate_raw(scn, device="cuda:0")
    lo, hi = scn.antenna_box(1e-3)
    plan = sar.Plan(scn.radar, scn.grid, scn.n_chirps, scn.n_rx, (lo, hi))
    tx = torch.as_tensor(scn.tx, device=dev)
    rx = None if scn.rx is None else torch.as_tensor(scn.rx, device=dev).contiguous()
    prof = plan.range_compress(raw, torch.as_tensor(scn.wsar, device=dev))
    img = plan.backproject(prof, tx, rx).cpu().numpy()
    r = scn.radar
    oprof = oracle.range_compress(raw.cpu().numpy(), r.fft_len, r.range_window, scn.wsar, k0=plan.k_lo, nk=plan.n_bins)
    img2 = plan.backproject(torch.as_tensor(oprof.astype(np.complex64), device=dev), tx, rx).cpu().numpy()
    ref = oracle.backproject(oprof, plan.k_lo, r, scn.tx, scn.rx, scn.grid.pixels()).reshape(img.shape)
    m = np.abs(ref).max()
    e1 = np.abs(img - ref); e2 = np.abs(img2 - ref)
    print(f"{tag}: full chain {e1.max()/m:.2e}  bp-only {e2.max()/m:.2e}  rc-diff {np.abs(prof.cpu().numpy()-oprof).max()/np.abs(oprof).max():.2e}")
    j, i = np.unravel_index(np.argmax(e2), e2.shape)
    print(f"   worst bp-only pixel (j,i)=({j},{i}) |ref|={abs(ref[j,i]):.3f} max|ref|={m:.3f} err={e2[j,i]:.3e}; tile-local ({j%32},{i%32})")
    # error vs distance from tile centre
    jj, ii = np.meshgrid(np.arange(img.shape[0]) % 32, np.arange(img.shape[1]) % 32, indexing="ij")
    rr = np.hypot(jj - 15.5, ii - 15.5)
    for lo_, hi_ in [(0, 6), (6, 12), (12, 18), (18, 23)]:
        sel = (rr >= lo_) & (rr < hi_)
        print(f"   |u| in [{lo_},{hi_}) px: mean err {e2[sel].mean()/m:.2e}  max {e2[sel].max()/m:.2e}")
    # error relative to local magnitude
    print(f"   median |err|/|ref| {np.median(e2/np.maximum(np.abs(ref),1e-9)):.2e}")
    plan.close()

run(sarsim.make_config("C1"), "C1")
run(sarsim.small_config(n_chirps=100, ns=256, nx=70, ny=90, seed=41), "small")
scn = sarsim.make_config("C1"); scn.radar = sarsim.Radar(n_samples=256, fft_len=2048, range_window=0)
run(scn, "C1-rect")
