"""Build libsar.so (the C-ABI CUDA library) in-tree with nvcc for sm_100a: every .cu compiled
to an object in parallel (the BP kernel families are separate translation units), then one
shared-library link with the static CUDA runtime."""
from __future__ import annotations

import concurrent.futures
import glob
import os
import subprocess
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsar.so")
CHECK_LIB = os.path.join(PKG, "libsar_check.so")   # -DSAR_DEBUG_CHECKS: bounds-check build (tests)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v"]
LDFLAGS = ARCH + ["-shared", "-cudart", "static"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu"))) + sorted(glob.glob(os.path.join(CSRC, "*.h"))) + \
        sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "sar_bp.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile and link; ``out``/``defines`` make tuning builds (tools/mkvariant.sh)."""
    out = out or LIB
    if out == LIB and not force and not stale():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with tempfile.TemporaryDirectory() as tmp:
        def compile_one(src):
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            cmd = [nvcc, *CFLAGS, *defines, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
            return obj, subprocess.run(cmd, capture_output=True, text=True)

        with concurrent.futures.ThreadPoolExecutor(max_workers=min(len(cu), os.cpu_count() or 4)) as ex:
            results = list(ex.map(compile_one, cu))
        log = ""
        for obj, res in results:
            log += res.stdout + res.stderr
            if res.returncode != 0:
                raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
        tmp_out = out + f".tmp{os.getpid()}"
        res = subprocess.run([nvcc, *LDFLAGS, "-o", tmp_out, *[o for o, _ in results]], capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
        os.replace(tmp_out, out)
    if out == LIB:
        with open(os.path.join(PKG, "build_ptxas.log"), "w") as f:
            f.write(log)
    if verbose:
        print(log)
    return out
