"""Incremental streaming SAR: continuous processing of a chirp stream
(a 1024-chirp measurement every N_m T_P0 = 109.3 ms; "even a continuous
SAR measurement could be processed without increasing delay").

With a world-fixed pixel grid, the image of an aperture of ``hops_per_frame`` hops is the
sum of per-hop partial images.  Each new hop costs one range compression of its chirps and
one back-projection of its chirps over the grid (into a ring slot); the frame is the sum of
the ring (``sar_image_sum``).  Per frame that is 1/hops_per_frame of the updates of the
sliding-window C5 frame.  Orchestration only: every step runs in libsar kernels.
"""
from __future__ import annotations

from . import sar


class IncrementalStream:
    def __init__(self, radar, grid, n_chirps_total: int, antenna_box, hop: int = 1024,
                 hops_per_frame: int = 8, device: int = 0, n_rx: int = 1):
        import torch

        self.plan = sar.Plan(radar, grid, n_chirps_total, n_rx, antenna_box, device=device)
        self.hop, self.k = hop, hops_per_frame
        self.dev = torch.device(f"cuda:{device}")
        self.ring = torch.zeros((hops_per_frame, grid.ny, grid.nx), dtype=torch.complex64, device=self.dev)
        self.frame = torch.zeros((grid.ny, grid.nx), dtype=torch.complex64, device=self.dev)
        self.prof = self.plan.empty_profiles()
        self.pushed = 0

    def push(self, raw, tx, rx=None, wsar=None, stream=None):
        """Process hop number ``self.pushed`` (chirps [h hop, (h+1) hop) of the full arrays)
        and return the current frame (sum of the last hops_per_frame partial images)."""
        h = self.pushed
        c0 = h * self.hop
        slot = h % self.k
        self.plan.range_compress(raw, wsar, chirp0=c0, nchirp=self.hop, out=self.prof, stream=stream)
        self.plan.backproject(self.prof, tx, rx, chirp0=c0, nchirp=self.hop, out=self.ring[slot], stream=stream)
        self.pushed += 1
        n = min(self.pushed, self.k)
        if n == self.k:
            sar.image_sum(self.ring, out=self.frame, stream=stream)
        else:
            sar.image_sum(self.ring[:n], out=self.frame, stream=stream)
        return self.frame

    def close(self):
        self.plan.close()
