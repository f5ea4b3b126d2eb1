"""Double-precision CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  The product path
(``paper_2306_09784_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle/sar_oracle.c`` (plain C, fp64, pthreads over
rows / pixels); this module only marshals numpy arrays through ctypes and
compiles the C file with gcc when the shared object is missing or stale.

Functions and the passages they follow (P:Lnnn = PAPER.md line):
  window            range window (reading A6)
  dft_row           literal range-compression sum, C-1 step 2
  fft               textbook radix-2 FFT (a library-primitive step)
  range_compress    H1, windowed zero-padded range FFT with centring ramp (A4-A8)
  backproject       H3-H5, Alg. 2 with Alg. 1 constants
  doppler_table     Measure D f_doppler(p) from the average velocity
  polar_to_cartesian  Measure E polar image -> Cartesian grid, bilinear
All are pinned by tests/test_oracle_pins.py (no function is "parity unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sar_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

C_LIGHT = 299792458.0


_STAMP = _LIB + ".cpu"


def _cpu_id() -> str:
    """The host CPU the library was tuned for (-march=native): model name + flags."""
    try:
        with open("/proc/cpuinfo") as f:
            txt = f.read()
        model = next((l.split(":", 1)[1].strip() for l in txt.splitlines() if l.startswith("model name")), "")
        flags = next((l.split(":", 1)[1].strip() for l in txt.splitlines() if l.startswith("flags")), "")
        return model + "|" + flags
    except OSError:
        return "unknown"


def build(force: bool = False) -> str:
    """Compile oracle/sar_oracle.c -> oracle/liboracle.so with gcc (no GPU needed): -O3
    -march=native as BASELINE.md's CPU-baseline plan states, FMA contraction off (the
    arithmetic stays the source's, operation by operation).  A library built for another
    host CPU (the tree travels to the GPU box) is rebuilt there."""
    stale = not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC)
    if not stale:
        try:
            with open(_STAMP) as f:
                stale = f.read() != _cpu_id()
        except OSError:
            stale = True
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O3", "-march=native", "-ffp-contract=off", "-std=c11", "-fPIC", "-shared", "-o", tmp, _SRC,
               "-lm", "-lpthread"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
        with open(_STAMP, "w") as f:
            f.write(_cpu_id())
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.POINTER
            d, i, f = ctypes.c_double, ctypes.c_int, ctypes.c_float
            lib.oracle_window.argtypes = [i, i, P(d)]
            lib.oracle_dft_row.argtypes = [P(d), i, i, P(d), d, i, i, P(d)]
            lib.oracle_fft.argtypes = [P(d), P(d), i]
            lib.oracle_range_compress.argtypes = [P(f), i, i, i, i, i, P(d), i, i, i, i, P(d)]
            lib.oracle_backproject.argtypes = [P(d), i, i, i, i, d, d, d, d, i,
                                               P(d), P(d), P(d), P(d), i, i, P(d)]
            lib.oracle_doppler_table.argtypes = [d, d, i, P(d), i, P(d), P(d), d, P(d)]
            lib.oracle_polar_to_cartesian.argtypes = [d, d, d, d, d, d, i, i, P(d), d, d, d, d, i, i, P(d)]
            for name in ("oracle_window", "oracle_dft_row", "oracle_fft", "oracle_doppler_table",
                         "oracle_polar_to_cartesian",
                         "oracle_range_compress", "oracle_backproject", "oracle_version"):
                getattr(lib, name).restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def _check(rc, what):
    if rc != 0:
        msg = {-1: "invalid argument", -2: "out of memory",
               -3: "profile crop does not cover a bin a pixel needs"}.get(rc, str(rc))
        raise RuntimeError(f"oracle {what} failed: {msg}")


def window(ns: int, kind: int = 1) -> np.ndarray:
    w = np.empty(ns, np.float64)
    _check(_load().oracle_window(ns, kind, _ptr(w, ctypes.c_double)), "window")
    return w


def dft_row(x, nfft: int, w, scale: float, k0: int, nk: int) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    w = np.ascontiguousarray(w, np.float64)
    out = np.empty((nk, 2), np.float64)
    _check(_load().oracle_dft_row(_ptr(x, ctypes.c_double), x.size, nfft, _ptr(w, ctypes.c_double),
                                  float(scale), k0, nk, _ptr(out, ctypes.c_double)), "dft_row")
    return out[:, 0] + 1j * out[:, 1]


def fft(z) -> np.ndarray:
    z = np.asarray(z, np.complex128)
    re = np.ascontiguousarray(z.real, np.float64).copy()
    im = np.ascontiguousarray(z.imag, np.float64).copy()
    _check(_load().oracle_fft(_ptr(re, ctypes.c_double), _ptr(im, ctypes.c_double), z.size), "fft")
    return re + 1j * im


def range_compress(raw, nfft: int, window_kind: int = 1, wsar=None, k0: int = 0,
                   nk: int | None = None, use_dft: bool = False, nthreads: int = 0) -> np.ndarray:
    """raw float32 [M][N_rx][Ns] -> complex128 profiles [M][N_rx][nk] of bins k0..k0+nk-1."""
    raw = np.ascontiguousarray(raw, np.float32)
    M, nrx, ns = raw.shape
    if nk is None:
        nk = nfft // 2 + 1 - k0
    ws = None if wsar is None else np.ascontiguousarray(wsar, np.float64)
    if ws is not None and ws.shape != (M,):
        raise ValueError("wsar must have one entry per chirp")
    out = np.empty((M, nrx, nk, 2), np.float64)
    _check(_load().oracle_range_compress(_ptr(raw, ctypes.c_float), M, nrx, ns, nfft, window_kind,
                                         _ptr(ws, ctypes.c_double), k0, nk, int(use_dft), nthreads,
                                         _ptr(out, ctypes.c_double)), "range_compress")
    return out[..., 0] + 1j * out[..., 1]


def backproject(prof, k0: int, radar, tx, rx, pixels, doppler=None, nthreads: int = 0) -> np.ndarray:
    """prof complex [M][N_rx][nk] (bins k0..), tx [M][3], rx [M][N_rx][3] or None (monostatic),
    pixels [P][3] -> complex128 [P].  ``radar`` needs f0_hz, bandwidth_hz, chirp_s,
    sample_rate_hz, fft_len."""
    prof = np.asarray(prof)
    M, nrx, nk = prof.shape
    pr = np.empty((M, nrx, nk, 2), np.float64)
    pr[..., 0] = prof.real
    pr[..., 1] = prof.imag
    tx = np.ascontiguousarray(tx, np.float64).reshape(M, 3)
    rxa = None if rx is None else np.ascontiguousarray(rx, np.float64).reshape(M, nrx, 3)
    pix = np.ascontiguousarray(pixels, np.float64).reshape(-1, 3)
    dop = None if doppler is None else np.ascontiguousarray(doppler, np.float64).reshape(-1)
    if dop is not None and dop.size != pix.shape[0]:
        raise ValueError("doppler must have one entry per pixel")
    out = np.empty((pix.shape[0], 2), np.float64)
    _check(_load().oracle_backproject(
        _ptr(pr, ctypes.c_double), M, nrx, k0, nk, float(radar.f0_hz), float(radar.bandwidth_hz),
        float(radar.chirp_s), float(radar.sample_rate_hz), int(radar.fft_len),
        _ptr(tx, ctypes.c_double), _ptr(rxa, ctypes.c_double), _ptr(dop, ctypes.c_double),
        _ptr(pix, ctypes.c_double), pix.shape[0], nthreads, _ptr(out, ctypes.c_double)), "backproject")
    return out[:, 0] + 1j * out[:, 1]


def doppler_table(radar, pixels, q_ref, v_avg, legs: float = 2.0) -> np.ndarray:
    """f_doppler(p) in bins for pixels [P][3] (Measure D)."""
    pix = np.ascontiguousarray(pixels, np.float64).reshape(-1, 3)
    q = np.ascontiguousarray(q_ref, np.float64).reshape(3)
    v = np.ascontiguousarray(v_avg, np.float64).reshape(3)
    out = np.empty(pix.shape[0], np.float64)
    _check(_load().oracle_doppler_table(float(radar.f0_hz), float(radar.sample_rate_hz), int(radar.fft_len),
                                        _ptr(pix, ctypes.c_double), pix.shape[0], _ptr(q, ctypes.c_double),
                                        _ptr(v, ctypes.c_double), float(legs), _ptr(out, ctypes.c_double)),
           "doppler_table")
    return out


def polar_to_cartesian(polar, img, cart) -> np.ndarray:
    """Polar image complex [n_r][n_th] of ``polar`` (xc, yc, r0, dr, th0, dth, n_th, n_r)
    -> complex128 [ny][nx] on Cartesian grid ``cart`` (x0, y0, dx, dy, nx, ny)."""
    img = np.asarray(img).reshape(polar.n_r, polar.n_th)
    src = np.empty((polar.n_r, polar.n_th, 2), np.float64)
    src[..., 0] = img.real
    src[..., 1] = img.imag
    out = np.empty((cart.ny, cart.nx, 2), np.float64)
    _check(_load().oracle_polar_to_cartesian(
        float(polar.xc), float(polar.yc), float(polar.r0), float(polar.dr), float(polar.th0), float(polar.dth),
        int(polar.n_th), int(polar.n_r), _ptr(src, ctypes.c_double), float(cart.x0), float(cart.y0),
        float(cart.dx), float(cart.dy), int(cart.nx), int(cart.ny), _ptr(out, ctypes.c_double)),
        "polar_to_cartesian")
    return out[..., 0] + 1j * out[..., 1]
