"""Derived-leg modes built by the BP producers on the scenes of tests/test_gpu_derived.py.

Run with the bounds-check build (SAR_LIB=paper_2306_09784_b200/libsar_check.so): prints one JSON
object {scene: [mono 2-term, mono 3-term, mono col 2, mono col 3, bi 3-term, bi 4-term, bi col 3,
bi col 4]} of group / stage counts (g_modes, reading A22)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import sarsim  # noqa: E402
from paper_2306_09784_b200 import sar  # noqa: E402

def make_scene(name):
    """The scenes (small_config geometry at 1 cm pixels, ~4.2-4.9 m range), tracks chosen so that
    the series bound (1e-9 m) selects one mode each."""
    kind, kw = SCENES[name]
    scn = sarsim.small_config(grid_dx=0.01, **kw)
    r = scn.radar
    if kind == "slow_straight":      # 0.2 mm steps
        scn.tx = sarsim.straight_track(scn.n_chirps, 0.2e-3)
    elif kind == "slow_curved":      # 1 -> 1.5 m/s on a 5 m arc (~0.1-0.16 mm steps)
        scn.tx = sarsim.curved_track(scn.n_chirps, r.pri_s, 1.0, 1.5, 5.0)
    if scn.rx is not None:
        scn.rx = sarsim.rx_array(scn.tx, scn.n_rx, 0.005, r.wavelength_m / 2.0)
    return scn


SCENES = {
    # monostatic, 0.2 mm steps: groups within the 2-term bound
    "mono_2term": ("slow_straight", dict(n_chirps=128, ns=256, nx=64, ny=64, seed=71)),
    # monostatic, curved track at 6 -> 9 m/s (~0.6-1 mm steps): the third term
    "mono_3term": ("as_is", dict(n_chirps=128, ns=256, nx=64, ny=64, seed=72, curved=True)),
    # 4-RX array along a straight track: collinear 3-term stages (compile-time 4 RX)
    "bi4_col3": ("slow_straight", dict(n_chirps=128, ns=256, nx=64, ny=64, seed=73, n_rx=4)),
    # 4-RX array on a slow arc: non-collinear 3-term stages
    "bi4_arc3": ("slow_curved", dict(n_chirps=128, ns=256, nx=64, ny=64, seed=74, n_rx=4)),
    # 4-RX array on the 6 -> 9 m/s arc: non-collinear 4-term stages
    "bi4_arc4": ("as_is", dict(n_chirps=128, ns=256, nx=64, ny=64, seed=76, n_rx=4, curved=True)),
    # 16-RX array (3.4 cm), straight: collinear 4-term stages, runtime RX count
    "bi16_col4": ("slow_straight", dict(n_chirps=64, ns=256, nx=64, ny=64, seed=75, n_rx=16)),
}
# modes (g_modes index) each scene must build: 0/1 mono 2/3 terms, 4/5 bistatic 3/4 terms,
# 6/7 bistatic collinear 3/4 terms
EXPECT = {"mono_2term": 0, "mono_3term": 1, "bi4_col3": 6, "bi4_arc3": 4, "bi4_arc4": 5, "bi16_col4": 7}


def modes(reset=True):
    lib = sar.load()
    f = getattr(lib, "sar_debug_modes_plain", None)
    if f is None:
        raise SystemExit("not a bounds-check build: SAR_LIB=paper_2306_09784_b200/libsar_check.so")
    buf = (ctypes.c_ulonglong * 8)()
    f(buf, int(reset))
    return list(buf)


if __name__ == "__main__":
    dev = torch.device("cuda:0")
    out = {}
    modes()
    for name in SCENES:
        scn = make_scene(name)
        raw = sarsim.simulate_raw(scn, device="cuda:0")
        lo, hi = scn.antenna_box(1e-3)
        p = sar.Plan(scn.radar, scn.grid, scn.n_chirps, scn.n_rx, (lo, hi))
        tx = torch.as_tensor(scn.tx, device=dev)
        rx = None if scn.rx is None else torch.as_tensor(scn.rx, device=dev).contiguous()
        p.backproject(p.range_compress(raw), tx, rx)
        torch.cuda.synchronize()
        out[name] = modes()
        p.close()
    print(json.dumps(out))
