"""Thin ctypes binding of libsar.so (include/sar_bp.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels
behind the C ABI.  There is no CPU fallback: if libsar.so is missing or cannot
be loaded this module raises.  Functions keep the C names; ``Plan`` is a small
convenience wrapper taking torch tensors (device memory and streams only).
"""
from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SAR_LIB", os.path.join(PKG, "libsar.so"))   # SAR_LIB: tuning builds

SAR_OK = 0
STATUS = {0: "SAR_OK", 1: "SAR_ERR_INVALID_ARGUMENT", 2: "SAR_ERR_OUT_OF_COVERAGE", 3: "SAR_ERR_CUDA",
          4: "SAR_ERR_NO_MEMORY", 5: "SAR_ERR_UNSUPPORTED_DEVICE"}


class SarError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class RadarParams(ctypes.Structure):
    _fields_ = [("f0_hz", ctypes.c_double), ("bandwidth_hz", ctypes.c_double), ("chirp_s", ctypes.c_double),
                ("pri_s", ctypes.c_double), ("sample_rate_hz", ctypes.c_double), ("n_samples", ctypes.c_int32),
                ("n_chirps", ctypes.c_int32), ("n_rx", ctypes.c_int32), ("fft_len", ctypes.c_int32),
                ("range_window", ctypes.c_int32), ("doppler_max_bins", ctypes.c_float)]


class Grid(ctypes.Structure):
    _fields_ = [("x0", ctypes.c_double), ("y0", ctypes.c_double), ("z0", ctypes.c_double),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("nx", ctypes.c_int32), ("ny", ctypes.c_int32)]


class PolarGrid(ctypes.Structure):
    _fields_ = [("xc", ctypes.c_double), ("yc", ctypes.c_double), ("zc", ctypes.c_double), ("r0", ctypes.c_double),
                ("dr", ctypes.c_double), ("th0", ctypes.c_double), ("dth", ctypes.c_double),
                ("n_th", ctypes.c_int32), ("n_r", ctypes.c_int32)]


class Box(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("chirp_rate_hz_per_s", ctypes.c_double), ("a1_bins_per_m", ctypes.c_double),
                ("c2_cycles_per_m", ctypes.c_double), ("d_min_m", ctypes.c_double), ("d_max_m", ctypes.c_double),
                ("k_lo", ctypes.c_int32), ("n_bins", ctypes.c_int32), ("tile_x", ctypes.c_int32),
                ("tile_y", ctypes.c_int32), ("window_bins", ctypes.c_int32), ("chirps_per_stage", ctypes.c_int32),
                ("updates_per_image", ctypes.c_int64), ("window_half_bins", ctypes.c_double),
                ("tile_rho_m", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None
_lock = threading.Lock()
P = ctypes.POINTER
_vp = ctypes.c_void_p
_i32 = ctypes.c_int32


def load() -> ctypes.CDLL:
    """Load libsar.so (raises if it was not built: run __graft_entry__.build())."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing; build it with __graft_entry__.build()")
            lib = ctypes.CDLL(LIB_PATH)
            lib.sar_plan_geometry.argtypes = [P(RadarParams), P(Grid), P(Box), P(PlanInfo)]
            lib.sar_plan_create.argtypes = [P(RadarParams), P(Grid), P(Box), _i32, P(_vp)]
            lib.sar_plan_info.argtypes = [_vp, P(PlanInfo)]
            lib.sar_plan_crop.argtypes = [_vp, P(_i32), P(_i32)]
            lib.sar_range_compress.argtypes = [_vp, _vp, _vp, _i32, _i32, _vp, _vp]
            lib.sar_backproject.argtypes = [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _vp]
            lib.sar_backproject_scatter.argtypes = [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, P(_vp), _i32,
                                                    _i32, _vp]
            lib.sar_backproject_scatter.restype = ctypes.c_int
            lib.sar_backproject_tiles.argtypes = [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _vp]
            lib.sar_backproject_scatter_tiles.argtypes = [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, P(_vp),
                                                          _i32, _i32, _vp]
            lib.sar_plan_tiles.argtypes = [_vp, P(_i32), P(_i32)]
            for n in ("sar_backproject_tiles", "sar_backproject_scatter_tiles", "sar_plan_tiles"):
                getattr(lib, n).restype = ctypes.c_int
            lib.sar_form_image.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp]
            lib.sar_doppler_table.argtypes = [P(RadarParams), P(Grid), P(ctypes.c_double * 3),
                                              P(ctypes.c_double * 3), _vp, _vp]
            lib.sar_doppler_table.restype = ctypes.c_int
            lib.sar_doppler_table_polar.argtypes = [P(RadarParams), P(PolarGrid), P(ctypes.c_double * 3),
                                                    P(ctypes.c_double * 3), _vp, _vp]
            lib.sar_doppler_table_polar.restype = ctypes.c_int
            lib.sar_plan_create_polar.argtypes = [P(RadarParams), P(PolarGrid), P(Box), _i32, P(_vp)]
            lib.sar_plan_geometry_polar.argtypes = [P(RadarParams), P(PolarGrid), P(Box), P(PlanInfo)]
            lib.sar_polar_to_cartesian.argtypes = [P(PolarGrid), _vp, P(Grid), _vp, _vp]
            for n in ("sar_plan_create_polar", "sar_plan_geometry_polar", "sar_polar_to_cartesian"):
                getattr(lib, n).restype = ctypes.c_int
            lib.sar_image_sum.argtypes = [_vp, _vp, _i32, ctypes.c_int64, ctypes.c_int64, _vp]
            lib.sar_image_sum.restype = ctypes.c_int
            lib.sar_plan_launch_count.argtypes = [_vp]
            lib.sar_plan_launch_count.restype = ctypes.c_int64
            lib.sar_destroy.argtypes = [_vp]
            lib.sar_last_error.restype = ctypes.c_char_p
            lib.sar_version.restype = ctypes.c_char_p
            for n in ("sar_plan_geometry", "sar_plan_create", "sar_plan_info", "sar_plan_crop", "sar_range_compress",
                      "sar_backproject", "sar_form_image", "sar_destroy"):
                getattr(lib, n).restype = ctypes.c_int
            _lib = lib
    return _lib


def _check(st: int):
    if st != SAR_OK:
        raise SarError(st, load().sar_last_error().decode())


# ------------------------------------------------------------------- C-named functions
def sar_plan_geometry(radar: RadarParams, grid: Grid, box: Box) -> PlanInfo:
    info = PlanInfo()
    _check(load().sar_plan_geometry(ctypes.byref(radar), ctypes.byref(grid), ctypes.byref(box), ctypes.byref(info)))
    return info


def sar_plan_create(radar: RadarParams, grid: Grid, box: Box, device: int = 0) -> int:
    h = _vp()
    _check(load().sar_plan_create(ctypes.byref(radar), ctypes.byref(grid), ctypes.byref(box), device, ctypes.byref(h)))
    return h.value


def sar_plan_create_polar(radar: RadarParams, grid: PolarGrid, box: Box, device: int = 0) -> int:
    h = _vp()
    _check(load().sar_plan_create_polar(ctypes.byref(radar), ctypes.byref(grid), ctypes.byref(box), device,
                                        ctypes.byref(h)))
    return h.value


def sar_plan_geometry_polar(radar: RadarParams, grid: PolarGrid, box: Box) -> PlanInfo:
    info = PlanInfo()
    _check(load().sar_plan_geometry_polar(ctypes.byref(radar), ctypes.byref(grid), ctypes.byref(box),
                                          ctypes.byref(info)))
    return info


def sar_polar_to_cartesian(polar: PolarGrid, polar_ptr, cart: Grid, out_ptr, stream=0):
    _check(load().sar_polar_to_cartesian(ctypes.byref(polar), polar_ptr, ctypes.byref(cart), out_ptr, stream))


def polar_grid_params(g) -> PolarGrid:
    return PolarGrid(g.xc, g.yc, g.zc, g.r0, g.dr, g.th0, g.dth, g.n_th, g.n_r)


def polar_to_cartesian(polar_grid, polar_img, cart_grid, out=None, stream=None):
    """Bilinear (bearing, range) resampling of a polar image onto a Cartesian grid."""
    import torch

    out = torch.empty((cart_grid.ny, cart_grid.nx), dtype=torch.complex64, device=polar_img.device) \
        if out is None else out
    sar_polar_to_cartesian(polar_grid_params(polar_grid),
                           _dptr(polar_img, torch.complex64, (polar_grid.n_r, polar_grid.n_th), "polar image"),
                           grid_params(cart_grid), _dptr(out, torch.complex64, (cart_grid.ny, cart_grid.nx), "out"),
                           _stream_handle(stream))
    return out


def sar_plan_info(plan: int) -> PlanInfo:
    info = PlanInfo()
    _check(load().sar_plan_info(plan, ctypes.byref(info)))
    return info


def sar_plan_crop(plan: int):
    k, n = _i32(), _i32()
    _check(load().sar_plan_crop(plan, ctypes.byref(k), ctypes.byref(n)))
    return k.value, n.value


def sar_range_compress(plan, raw_ptr, wsar_ptr, chirp0, nchirp, prof_ptr, stream=0):
    _check(load().sar_range_compress(plan, raw_ptr, wsar_ptr, chirp0, nchirp, prof_ptr, stream))


def sar_backproject(plan, prof_ptr, tx_ptr, rx_ptr, dop_ptr, chirp0, nchirp, row0, nrow, img_ptr,
                    accumulate=0, stream=0):
    _check(load().sar_backproject(plan, prof_ptr, tx_ptr, rx_ptr, dop_ptr, chirp0, nchirp, row0, nrow,
                                  img_ptr, accumulate, stream))


SAR_SCATTER_MULTICAST = 1
SAR_SCATTER_ADD = 2
SAR_SCATTER_PUBLISH = 4   # sar_backproject_scatter_tiles: compute into images[0], then copy to the others


def sar_backproject_scatter(plan, prof_ptr, tx_ptr, rx_ptr, dop_ptr, chirp0, nchirp, row0, nrow, image_ptrs,
                            flags=0, stream=0):
    arr = (_vp * len(image_ptrs))(*image_ptrs)
    _check(load().sar_backproject_scatter(plan, prof_ptr, tx_ptr, rx_ptr, dop_ptr, chirp0, nchirp, row0, nrow,
                                          arr, len(image_ptrs), int(flags), stream))


def sar_backproject_tiles(plan, prof_ptr, tx_ptr, rx_ptr, dop_ptr, chirp0, nchirp, tile0, ntile, img_ptr,
                          accumulate=0, stream=0):
    _check(load().sar_backproject_tiles(plan, prof_ptr, tx_ptr, rx_ptr, dop_ptr, chirp0, nchirp, tile0, ntile,
                                        img_ptr, accumulate, stream))


def sar_backproject_scatter_tiles(plan, prof_ptr, tx_ptr, rx_ptr, dop_ptr, chirp0, nchirp, tile0, ntile,
                                  image_ptrs, flags=0, stream=0):
    arr = (_vp * len(image_ptrs))(*image_ptrs)
    _check(load().sar_backproject_scatter_tiles(plan, prof_ptr, tx_ptr, rx_ptr, dop_ptr, chirp0, nchirp, tile0,
                                                ntile, arr, len(image_ptrs), int(flags), stream))


def sar_plan_tiles(plan):
    tx, ty = _i32(), _i32()
    _check(load().sar_plan_tiles(plan, ctypes.byref(tx), ctypes.byref(ty)))
    return tx.value, ty.value


def sar_form_image(plan, raw_h, wsar_h, tx_h, rx_h, dop_h, row0, nrow, img_h, stream=0):
    _check(load().sar_form_image(plan, raw_h, wsar_h, tx_h, rx_h, dop_h, row0, nrow, img_h, stream))


def sar_doppler_table(radar: RadarParams, grid: Grid, q_ref, v_avg, dop_ptr, stream=0):
    q = (ctypes.c_double * 3)(*[float(v) for v in q_ref])
    v = (ctypes.c_double * 3)(*[float(x) for x in v_avg])
    _check(load().sar_doppler_table(ctypes.byref(radar), ctypes.byref(grid), ctypes.byref(q), ctypes.byref(v),
                                    dop_ptr, stream))


def doppler_bound_bins(radar, v_avg) -> float:
    """|f_doppler| <= 2 f0 |v_avg| N / (c fs): a valid doppler_max_bins for a plan."""
    import math

    speed = math.sqrt(sum(float(x) ** 2 for x in v_avg))
    return 2.0 * radar.f0_hz * speed / 299792458.0 * radar.fft_len / radar.sample_rate_hz


def sar_doppler_table_polar(radar: RadarParams, grid: PolarGrid, q_ref, v_avg, dop_ptr, stream=0):
    q = (ctypes.c_double * 3)(*[float(v) for v in q_ref])
    v = (ctypes.c_double * 3)(*[float(x) for x in v_avg])
    _check(load().sar_doppler_table_polar(ctypes.byref(radar), ctypes.byref(grid), ctypes.byref(q), ctypes.byref(v),
                                          dop_ptr, stream))


def doppler_table(radar, grid, q_ref, v_avg, device=0, out=None, stream=None):
    """Measure D table (float32 [ny][nx], CUDA) via sar_doppler_table (polar grids: [n_r][n_th]
    via sar_doppler_table_polar)."""
    import torch

    out = torch.empty((grid.ny, grid.nx), dtype=torch.float32, device=f"cuda:{device}") if out is None else out
    ptr = _dptr(out, torch.float32, (grid.ny, grid.nx), "doppler")
    if hasattr(grid, "n_th"):
        sar_doppler_table_polar(radar_params(radar, 1, 1), polar_grid_params(grid), q_ref, v_avg, ptr,
                                _stream_handle(stream))
    else:
        sar_doppler_table(radar_params(radar, 1, 1), grid_params(grid), q_ref, v_avg, ptr, _stream_handle(stream))
    return out


def sar_image_sum(out_ptr, partials_ptr, n_partials, stride, n_elems, stream=0):
    _check(load().sar_image_sum(out_ptr, partials_ptr, n_partials, stride, n_elems, stream))


def image_sum(partials, out=None, stream=None):
    """out = partials.sum(0) in k order, partials complex64 CUDA [n][...] (sar_image_sum)."""
    import torch

    n = partials.shape[0]
    per = partials[0].numel()
    out = torch.empty(partials.shape[1:], dtype=torch.complex64, device=partials.device) if out is None else out
    sar_image_sum(_dptr(out, torch.complex64, tuple(partials.shape[1:]), "out"),
                  _dptr(partials, torch.complex64, None, "partials"), n, per, per, _stream_handle(stream))
    return out


def sar_plan_launch_count(plan) -> int:
    return int(load().sar_plan_launch_count(plan))


def sar_destroy(plan):
    _check(load().sar_destroy(plan))


def sar_version() -> str:
    return load().sar_version().decode()


# ------------------------------------------------------------------- torch-facing wrapper
def radar_params(radar, n_chirps: int, n_rx: int, doppler_max_bins: float = 0.0) -> RadarParams:
    """From any object with the Table 1 fields (e.g. sarsim.Radar)."""
    return RadarParams(radar.f0_hz, radar.bandwidth_hz, radar.chirp_s, radar.pri_s, radar.sample_rate_hz,
                       radar.n_samples, n_chirps, n_rx, radar.fft_len, radar.range_window, doppler_max_bins)


def grid_params(g) -> Grid:
    return Grid(g.x0, g.y0, g.z0, g.dx, g.dy, g.nx, g.ny)


def box_params(lo, hi) -> Box:
    b = Box()
    for k in range(3):
        b.lo[k] = float(lo[k])
        b.hi[k] = float(hi[k])
    return b


def _stream_handle(stream) -> int:
    if stream is None:
        import torch

        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _dptr(t, dtype, shape=None, name="tensor"):
    import torch

    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    return t.data_ptr()


def _hptr(t, dtype, shape, name):
    import torch

    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous host {dtype} tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}")
    return t.data_ptr()


class Plan:
    """Owns a sar_plan_t.  Tensors in, tensors out; all work on the given CUDA stream."""

    def __init__(self, radar, grid, n_chirps: int, n_rx: int, antenna_box, device: int = 0,
                 doppler_max_bins: float = 0.0):
        self.radar = radar
        self.grid = grid
        self.n_chirps = n_chirps
        self.n_rx = n_rx
        self.device = device
        self._rp = radar_params(radar, n_chirps, n_rx, doppler_max_bins)
        self._bp = box_params(*antenna_box)
        self.polar = hasattr(grid, "n_th")     # a polar grid (sarsim.PolarGrid): image [n_r][n_th]
        if self.polar:
            self._gp = polar_grid_params(grid)
            self.handle = sar_plan_create_polar(self._rp, self._gp, self._bp, device)
        else:
            self._gp = grid_params(grid)
            self.handle = sar_plan_create(self._rp, self._gp, self._bp, device)
        self.info = sar_plan_info(self.handle)
        self.k_lo, self.n_bins = self.info.k_lo, self.info.n_bins

    def close(self):
        if getattr(self, "handle", None):
            sar_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- allocation helpers (torch for device memory)
    def empty_profiles(self):
        import torch

        return torch.empty((self.n_chirps, self.n_rx, self.n_bins), dtype=torch.complex64, device=f"cuda:{self.device}")

    def empty_image(self, nrow=None):
        import torch

        nrow = self.grid.ny if nrow is None else nrow
        return torch.empty((nrow, self.grid.nx), dtype=torch.complex64, device=f"cuda:{self.device}")

    def range_compress(self, raw, wsar=None, chirp0=0, nchirp=None, out=None, stream=None):
        import torch

        nchirp = self.n_chirps - chirp0 if nchirp is None else nchirp
        out = self.empty_profiles() if out is None else out
        sar_range_compress(self.handle, _dptr(raw, torch.float32, (self.n_chirps, self.n_rx, self.radar.n_samples), "raw"),
                           _dptr(wsar, torch.float32, (self.n_chirps,), "wsar"), chirp0, nchirp,
                           _dptr(out, torch.complex64, (self.n_chirps, self.n_rx, self.n_bins), "profiles"),
                           _stream_handle(stream))
        return out

    def backproject(self, profiles, tx, rx=None, doppler=None, chirp0=0, nchirp=None, row0=0, nrow=None,
                    out=None, accumulate=False, stream=None):
        import torch

        nchirp = self.n_chirps - chirp0 if nchirp is None else nchirp
        nrow = self.grid.ny - row0 if nrow is None else nrow
        out = self.empty_image(nrow) if out is None else out
        sar_backproject(self.handle,
                        _dptr(profiles, torch.complex64, (self.n_chirps, self.n_rx, self.n_bins), "profiles"),
                        _dptr(tx, torch.float64, (self.n_chirps, 3), "tx"),
                        _dptr(rx, torch.float64, (self.n_chirps, self.n_rx, 3), "rx"),
                        _dptr(doppler, torch.float32, (self.grid.ny, self.grid.nx), "doppler"),
                        chirp0, nchirp, row0, nrow,
                        _dptr(out, torch.complex64, (nrow, self.grid.nx), "image"), int(bool(accumulate)),
                        _stream_handle(stream))
        return out

    def backproject_scatter(self, profiles, tx, image_ptrs, rx=None, doppler=None, chirp0=0, nchirp=None, row0=0,
                            nrow=None, multicast=False, add=False, stream=None):
        """Back-project rows [row0, row0+nrow) and store (``add``: atomically add) each finished tile
        at its absolute rows of every full image in ``image_ptrs`` (device addresses: local,
        P2P-mapped peer buffers, or one multicast address with ``multicast=True``) -- the gather
        (or the chirp-shard reduction) fused into the epilogue."""
        import torch

        nchirp = self.n_chirps - chirp0 if nchirp is None else nchirp
        nrow = self.grid.ny - row0 if nrow is None else nrow
        sar_backproject_scatter(self.handle,
                                _dptr(profiles, torch.complex64, (self.n_chirps, self.n_rx, self.n_bins), "profiles"),
                                _dptr(tx, torch.float64, (self.n_chirps, 3), "tx"),
                                _dptr(rx, torch.float64, (self.n_chirps, self.n_rx, 3), "rx"),
                                _dptr(doppler, torch.float32, (self.grid.ny, self.grid.nx), "doppler"),
                                chirp0, nchirp, row0, nrow, [int(p) for p in image_ptrs],
                                (SAR_SCATTER_MULTICAST if multicast else 0) | (SAR_SCATTER_ADD if add else 0),
                                _stream_handle(stream))

    @property
    def tiles(self):
        """(tiles_x, tiles_y): the absolute BP tile grid (tile t = ty * tiles_x + tx)."""
        return sar_plan_tiles(self.handle)

    def backproject_tiles(self, profiles, tx, tile0, ntile, rx=None, doppler=None, chirp0=0, nchirp=None, out=None,
                          accumulate=False, stream=None):
        """Back-project the absolute tiles [tile0, tile0+ntile) into the FULL image ``out``
        ([ny][nx]; only those tiles' pixels are written)."""
        import torch

        g = self.grid
        nchirp = self.n_chirps - chirp0 if nchirp is None else nchirp
        out = self.empty_image() if out is None else out
        sar_backproject_tiles(self.handle,
                              _dptr(profiles, torch.complex64, (self.n_chirps, self.n_rx, self.n_bins), "profiles"),
                              _dptr(tx, torch.float64, (self.n_chirps, 3), "tx"),
                              _dptr(rx, torch.float64, (self.n_chirps, self.n_rx, 3), "rx"),
                              _dptr(doppler, torch.float32, (g.ny, g.nx), "doppler"),
                              chirp0, nchirp, tile0, ntile, _dptr(out, torch.complex64, (g.ny, g.nx), "image"),
                              int(bool(accumulate)), _stream_handle(stream))
        return out

    def backproject_scatter_tiles(self, profiles, tx, image_ptrs, tile0, ntile, rx=None, doppler=None, chirp0=0,
                                  nchirp=None, multicast=False, add=False, publish=False, stream=None):
        """``backproject_scatter`` over the absolute tiles [tile0, tile0+ntile); ``publish``:
        compute into image_ptrs[0] (the caller's own image), then copy the tiles to the others
        (SAR_SCATTER_PUBLISH)."""
        import torch

        g = self.grid
        nchirp = self.n_chirps - chirp0 if nchirp is None else nchirp
        sar_backproject_scatter_tiles(self.handle,
                                      _dptr(profiles, torch.complex64, (self.n_chirps, self.n_rx, self.n_bins),
                                            "profiles"),
                                      _dptr(tx, torch.float64, (self.n_chirps, 3), "tx"),
                                      _dptr(rx, torch.float64, (self.n_chirps, self.n_rx, 3), "rx"),
                                      _dptr(doppler, torch.float32, (g.ny, g.nx), "doppler"),
                                      chirp0, nchirp, tile0, ntile, [int(p) for p in image_ptrs],
                                      (SAR_SCATTER_MULTICAST if multicast else 0) | (SAR_SCATTER_ADD if add else 0)
                                      | (SAR_SCATTER_PUBLISH if publish else 0),
                                      _stream_handle(stream))

    def form_image(self, raw_h, tx_h, rx_h=None, wsar_h=None, doppler_h=None, row0=0, nrow=None, out_h=None,
                   stream=None, sync=True):
        """End-to-end from host tensors (pinned for async copies): image rows [row0, row0+nrow)."""
        import torch

        g = self.grid
        nrow = g.ny - row0 if nrow is None else nrow
        out_h = torch.empty((nrow, g.nx), dtype=torch.complex64, pin_memory=True) if out_h is None else out_h
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        sar_form_image(self.handle,
                       _hptr(raw_h, torch.float32, (self.n_chirps, self.n_rx, self.radar.n_samples), "raw_h"),
                       _hptr(wsar_h, torch.float32, (self.n_chirps,), "wsar_h"),
                       _hptr(tx_h, torch.float64, (self.n_chirps, 3), "tx_h"),
                       _hptr(rx_h, torch.float64, (self.n_chirps, self.n_rx, 3), "rx_h"),
                       _hptr(doppler_h, torch.float32, (g.ny, g.nx), "doppler_h"), row0, nrow,
                       _hptr(out_h, torch.complex64, (nrow, g.nx), "image_h"), int(st.cuda_stream))
        if sync:
            st.synchronize()
        return out_h

    @property
    def launches(self) -> int:
        return sar_plan_launch_count(self.handle)
