# compute-sanitizer availability probe on a tiny BP (C1-sized)
which compute-sanitizer; compute-sanitizer --version | head -2
cat > /tmp/tiny.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, sarsim
from paper_2306_09784_b200 import sar
scn = sarsim.small_config(n_chirps=32, ns=128, nx=40, ny=24, n_rx=2, seed=3)
raw = sarsim.simulate_raw(scn, device="cuda:0")
lo, hi = scn.antenna_box(1e-3)
p = sar.Plan(scn.radar, scn.grid, scn.n_chirps, scn.n_rx, (lo, hi))
tx = torch.as_tensor(scn.tx, device="cuda:0"); rx = torch.as_tensor(scn.rx, device="cuda:0").contiguous()
img = p.backproject(p.range_compress(raw), tx, rx); torch.cuda.synchronize(); print("ok", float(img.abs().max()))
PY
timeout 600 compute-sanitizer --tool memcheck --target-processes all python /tmp/tiny.py 2>&1 | tail -8
