"""B200-native FMCW range compression + time-domain Back-Projection (arXiv 2306.09784).

The product is ``libsar.so`` (C ABI, include/sar_bp.h) built from ``csrc/``;
``sar`` is its thin ctypes binding and ``dist`` the torch.distributed sharding
helpers (pixel rows -> all-gather, chirps -> reduce).
"""

__all__ = ["sar", "dist"]
