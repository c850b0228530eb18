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
# adaln_capi.cu (C ABI, planning, launches) + one kernel-instantiation TU per dtype, compiled in
# parallel and linked into one library (tools/gen_instances.py writes the instance lists)
SOURCES = ["adaln_capi.cu", "instances_f32.cu", "instances_bf16.cu", "instances_f16.cu",
           "instances_f64.cu"]
HEADERS = ["adaln_kernels.cuh", "bwd_steal.cuh", "block_kernels.cuh", "dtype.cuh", "ptx.cuh",
           "instances_extern.inc"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-diag-suppress", "20279,20281"]


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
    objdir = LIBDIR / "obj"
    objdir.mkdir(exist_ok=True)
    nvcc = _nvcc()
    procs = []
    for src in SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        cmd = [nvcc, ARCH, *FLAGS, "-Xptxas", "-v", "-c", "-o", str(obj), str(CSRC / src)]
        procs.append((src, obj, subprocess.Popen(cmd, cwd=str(CSRC), stdout=subprocess.PIPE,
                                                 stderr=subprocess.PIPE, text=True)))
    logs, failed = [], []
    for src, _, pr in procs:
        out, err = pr.communicate()
        logs.append(f"==== {src}\n{out}{err}")
        if pr.returncode != 0:
            failed.append(f"{src}:\n{err[-3000:]}")
    (LIBDIR / "ptxas.log").write_text("\n".join(logs))
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(failed))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, ARCH, "--shared", "-cudart", "static", "-o", str(tmp)] + [str(o) for _, o, _ in procs]
    proc = subprocess.run(cmd, cwd=str(CSRC), capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({proc.returncode}):\n{proc.stderr[-4000:]}")
    if verbose:
        print(logs[0][-2000:])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build_native(force=True, verbose=False))
