import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, sarsim, oracle
from sarsim import Scenario
from tests.helpers import gpu_image, oracle_image, rel_err
scn = sarsim.small_config(n_chirps=96, ns=256, nx=40, ny=30, curved=True, n_rx=2, seed=32)
raw = sarsim.simulate_raw(scn, device="cuda:0")
ref0 = oracle_image(scn, raw.cpu().numpy())
for rep in range(3):
    a = gpu_image(scn, raw).cpu().numpy().reshape(-1)
    print("unperm rep", rep, "err", rel_err(a, ref0), "max", np.abs(a).max(), flush=True)
perm = np.random.default_rng(2).permutation(96)
scn2 = Scenario("perm", scn.radar, scn.grid, scn.tx[perm], scn.rx[perm], scn.targets, scn.amps, scn.isolated, scn.wsar[perm])
raw2 = raw[perm.tolist()].contiguous()
b = gpu_image(scn2, raw2).cpu().numpy().reshape(-1)
print("perm rel err vs oracle", rel_err(b, ref0), "vs a", rel_err(b, a), flush=True)
