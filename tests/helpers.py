"""Shared helpers for the parity tests: run the CUDA path through the C ABI, run the
oracle on the same seeded inputs, compare with the north-star bar."""
from __future__ import annotations

import numpy as np

import oracle
import sarsim

REL_TOL = 1e-3   # north star: max|img_gpu - img_ref| / max|img_ref| <= 1e-3


def gpu_image(scn, raw=None, device=0, row0=0, nrow=None, doppler=None, dop_max=0.0, return_prof=False,
              plan=None, box_margin=1e-3):
    import torch

    from paper_2306_09784_b200 import sar

    dev = torch.device(f"cuda:{device}")
    if raw is None:
        raw = sarsim.simulate_raw(scn, device=str(dev))
    raw = raw.to(dev)
    lo, hi = scn.antenna_box(box_margin)
    own = plan is None
    if own:
        plan = sar.Plan(scn.radar, scn.grid, scn.n_chirps, scn.n_rx, (lo, hi), device=device,
                        doppler_max_bins=dop_max)
    tx = torch.as_tensor(scn.tx, device=dev)
    rx = None if scn.rx is None else torch.as_tensor(scn.rx, device=dev).contiguous()
    wsar = torch.as_tensor(scn.wsar, device=dev)
    prof = plan.range_compress(raw, wsar)
    dop = None if doppler is None else torch.as_tensor(doppler, dtype=torch.float32, device=dev).contiguous()
    img = plan.backproject(prof, tx, rx, dop, row0=row0, nrow=nrow)
    torch.cuda.synchronize()
    out = (img, prof, plan) if return_prof else img
    if own and not return_prof:
        plan.close()
    return out


def oracle_profiles(scn, raw_np, k_lo=0, n_bins=None, nthreads=0):
    r = scn.radar
    return oracle.range_compress(raw_np, r.fft_len, r.range_window, scn.wsar, k0=k_lo, nk=n_bins,
                                 nthreads=nthreads)


def oracle_image(scn, raw_np, pixels=None, doppler=None, nthreads=0):
    prof = oracle_profiles(scn, raw_np, nthreads=nthreads)
    pix = scn.grid.pixels() if pixels is None else pixels
    return oracle.backproject(prof, 0, scn.radar, scn.tx, scn.rx, pix, doppler, nthreads=nthreads)


def rel_err(got, ref):
    got = np.asarray(got, np.complex128)
    ref = np.asarray(ref, np.complex128)
    return float(np.abs(got - ref).max() / np.abs(ref).max())


def sample_indices(scn, gpu_abs=None, stride=(97, 101), win=3, top=32):
    """C-6 protocol: strided rows/cols + +-win windows around isolated targets and the
    GPU's top local maxima.  Returns unique (j, i) pairs."""
    g = scn.grid
    js = np.arange(0, g.ny, stride[0])
    iis = np.arange(0, g.nx, stride[1])
    pts = [np.stack(np.meshgrid(js, iis, indexing="ij"), -1).reshape(-1, 2)]
    centres = [tuple(c) for c in scn.isolated]
    if gpu_abs is not None:
        flat = np.argsort(gpu_abs.reshape(-1))[::-1][:top]
        centres += [tuple(np.unravel_index(f, gpu_abs.shape)) for f in flat]
    d = np.arange(-win, win + 1)
    for (j, i) in centres:
        jj, ii = np.meshgrid(j + d, i + d, indexing="ij")
        w = np.stack([jj, ii], -1).reshape(-1, 2)
        ok = (w[:, 0] >= 0) & (w[:, 0] < g.ny) & (w[:, 1] >= 0) & (w[:, 1] < g.nx)
        pts.append(w[ok])
    allp = np.concatenate(pts)
    return np.unique(allp, axis=0)


def c6_indices(scn, gpu_abs, stride=31, win=24, top=32):
    """The C-6 protocol: WHOLE grid rows and columns at ``stride`` (coprime with the
    32-px tile, so every tile row / column offset is visited), the last (ragged) row and column,
    and +-``win`` px windows around every isolated target and the GPU's ``top`` largest pixels.
    Returns unique (j, i) pairs."""
    g = scn.grid
    rows = np.unique(np.r_[np.arange(0, g.ny, stride), g.ny - 1])
    cols = np.unique(np.r_[np.arange(0, g.nx, stride), g.nx - 1])
    pts = [np.stack(np.meshgrid(rows, np.arange(g.nx), indexing="ij"), -1).reshape(-1, 2),
           np.stack(np.meshgrid(np.arange(g.ny), cols, indexing="ij"), -1).reshape(-1, 2)]
    centres = [tuple(c) for c in scn.isolated]
    flat = np.argsort(gpu_abs.reshape(-1))[::-1][:top]
    centres += [tuple(np.unravel_index(f, gpu_abs.shape)) for f in flat]
    d = np.arange(-win, win + 1)
    for (j, i) in centres:
        jj, ii = np.meshgrid(j + d, i + d, indexing="ij")
        w = np.stack([jj, ii], -1).reshape(-1, 2)
        ok = (w[:, 0] >= 0) & (w[:, 0] < g.ny) & (w[:, 1] >= 0) & (w[:, 1] < g.nx)
        pts.append(w[ok])
    return np.unique(np.concatenate(pts), axis=0)
