"""Build the in-tree native libraries.

* ``_lib/libadaln_b200.so`` -- the sm_100a CUDA kernels + C ABI (``include/adaln_b200.h``),
  compiled by nvcc directly (no torch extension machinery: the ABI carries no torch types).

The .so is written into the package directory so it travels with the repo snapshot to the GPU
box; nothing is cached under ``~/.cache``.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libadaln_b200.so"

ARCH = "-gencode=arch=compute_100a,code=sm_100a"
SOURCES = ["adaln_capi.cu"]
HEADERS = ["adaln_kernels.cuh", "block_kernels.cuh", "dtype.cuh", "ptx.cuh"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; cannot build the sm_100a AdaLN library")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_native(force: bool = False, verbose: bool = False) -> Path:
    """Compile ``libadaln_b200.so`` for sm_100a if it is missing or older than its sources."""
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "adaln_b200.h"]
    if not force and not _stale(LIB, deps):
        return LIB
    LIBDIR.mkdir(exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [
        _nvcc(), ARCH, "-O3", "-lineinfo", "-std=c++17", "--shared", "-Xcompiler", "-fPIC",
        "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v", "--expt-relaxed-constexpr",
        "-cudart", "static", "-o", str(tmp),
    ] + [str(CSRC / s) for s in SOURCES]
    proc = subprocess.run(cmd, cwd=str(CSRC), capture_output=True, text=True)
    (LIBDIR / "ptxas.log").write_text(proc.stdout + proc.stderr)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{proc.stderr[-4000:]}")
    if verbose:
        print(proc.stderr[-2000:])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build_native(force=True, verbose=False))
