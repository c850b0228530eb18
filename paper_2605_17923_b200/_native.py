"""ctypes binding of ``libadaln_b200.so`` (the C ABI declared in ``include/adaln_b200.h``).

This is the same stub a maintainer of the reference would add: plain
pointers and sizes, no torch types.  There is no fallback: if the library is missing or a call
fails, an exception is raised.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import InvalidTile, NativeLibraryError, ShapeMismatch

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libadaln_b200.so"
# A/B hook for kernel experiments (tools/ab_variant.sh): load another in-tree build instead
if os.environ.get("AL_LIB_VARIANT"):
    LIB_PATH = LIB_PATH.parent / "variants" / (os.environ["AL_LIB_VARIANT"] + ".so")

AL_OK = 0
AL_ERR_SHAPE = 1
AL_ERR_TILE = 3
AL_ERR_VALUE = 5
AL_ERR_DTYPE = 6
AL_ERR_WORKSPACE = 7
AL_ERR_CUDA = 8

AL_F32, AL_BF16, AL_F16, AL_F64 = 0, 1, 2, 3

AL_BWD_DETERMINISTIC = 1  # al_adaln_backward flags

ABI_VERSION = 5

# every symbol include/adaln_b200.h declares: (name, restype, argtypes)
_i64 = ctypes.c_int64
_p = ctypes.c_void_p
_SIGNATURES = {
    "al_abi_version": (ctypes.c_int, []),
    "al_last_error": (ctypes.c_char_p, []),
    "al_device_init": (ctypes.c_int, [ctypes.c_int]),
    "al_adaln_forward": (
        ctypes.c_int,
        [_p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, ctypes.c_int, ctypes.c_double, _p, _p],
    ),
    "al_adaln_gate_residual_forward": (
        ctypes.c_int,
        [_p, _p, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, ctypes.c_int,
         ctypes.c_double, _p, _p],
    ),
    "al_gate_residual_backward_workspace_bytes": (_i64, [_i64, _i64, _i64, _i64, ctypes.c_int]),
    "al_gate_residual_backward": (
        ctypes.c_int,
        [_p, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, ctypes.c_int, _p],
    ),
    "al_qk_rmsnorm_forward": (
        ctypes.c_int,
        [_p, _i64, _p, _p, _p, _p, _p, _p, _i64, _i64, ctypes.c_int, ctypes.c_double, _p, _p],
    ),
    "al_qk_rmsnorm_backward_workspace_bytes": (_i64, [_i64, _i64, ctypes.c_int]),
    "al_qk_rmsnorm_backward": (
        ctypes.c_int,
        [_p, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, ctypes.c_int, _p, _p],
    ),
    "al_adaln_backward_workspace_bytes": (_i64, [_i64, _i64, _i64, _i64, ctypes.c_int, _i64]),
    "al_adaln_backward": (
        ctypes.c_int,
        [_p, _p, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, ctypes.c_int,
         _i64, _i64, ctypes.c_int, _p, _p],
    ),
    "al_set_tuning": (ctypes.c_int, [ctypes.c_int] * 6),
    "al_debug_clock_probe": (ctypes.c_int, [_p, ctypes.c_uint, _p]),
    "al_debug_set_timestamps": (ctypes.c_int, [_p, ctypes.c_int]),
    "al_debug_steal_count": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_uint)]),
    "al_describe_launch": (
        ctypes.c_int,
        [ctypes.c_int, _i64, _i64, _i64, _i64, ctypes.c_int, _i64, ctypes.POINTER(_i64)],
    ),
}

_lib = None
_lock = threading.Lock()
_inited_devices: set[int] = set()


def load() -> ctypes.CDLL:
    """Load (once) and return the native library; raise NativeLibraryError if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeLibraryError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (nvcc, sm_100a). There is no CPU fallback."
            )
        try:
            lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
        except OSError as exc:  # pragma: no cover - depends on the box
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.al_abi_version() != ABI_VERSION:
            raise NativeLibraryError("libadaln_b200.so ABI version mismatch; rebuild it")
        _lib = lib
        return lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def last_error() -> str:
    msg = load().al_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    """Map a C status code onto the reference's exception types."""
    if rc == AL_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == AL_ERR_SHAPE:
        raise ShapeMismatch(msg)
    if rc == AL_ERR_TILE:
        raise InvalidTile(msg)
    if rc == AL_ERR_VALUE:
        raise ValueError(msg)
    raise NativeLibraryError(f"{msg} (status {rc})")


def ensure_device(device_index: int) -> None:
    """Load kernel images / set smem attributes once per device (outside any graph capture)."""
    if device_index in _inited_devices:
        return
    lib = load()
    import torch

    with torch.cuda.device(device_index):
        check(lib.al_device_init(device_index), "al_device_init")
    _inited_devices.add(device_index)


def set_tuning(kernel: int, vecs_per_thread: int = 0, rows_per_stage: int = 0,
               smem_budget: int = 0, force_generic: bool = False, variant: int = 0) -> None:
    check(load().al_set_tuning(kernel, vecs_per_thread, rows_per_stage, smem_budget,
                               int(force_generic), variant), "al_set_tuning")


def clock_probe(out_ptr: int, spin_ns: int, stream_ptr: int) -> None:
    """Enqueue the SM-clock probe (al_debug_clock_probe) writing 2 uint64 at out_ptr."""
    check(load().al_debug_clock_probe(out_ptr, spin_ns, stream_ptr), "al_debug_clock_probe")


def set_timestamps(buf_ptr: int | None, capacity: int = 0) -> None:
    """Route per-launch [start, end] device timestamps into a caller-initialised device buffer
    (al_debug_set_timestamps); None disables."""
    check(load().al_debug_set_timestamps(buf_ptr, capacity if buf_ptr else 0),
          "al_debug_set_timestamps")


def steal_count(slot: int = 0) -> int:
    """Chunks stolen so far on work-stealing protocol slot `slot` (al_debug_steal_count)."""
    v = ctypes.c_uint(0)
    check(load().al_debug_steal_count(slot, ctypes.byref(v)), "al_debug_steal_count")
    return int(v.value)


def describe_launch(kernel: int, batch: int, seq: int, dim: int, mod_stride: int, dtype: int,
                    n_tile: int = 0) -> dict:
    out = (_i64 * 7)()
    check(load().al_describe_launch(kernel, batch, seq, dim, mod_stride, dtype, n_tile, out),
          "al_describe_launch")
    keys = ("path", "grid", "threads", "vecs_per_thread", "rows_per_stage", "stages", "smem_bytes")
    d = dict(zip(keys, list(out)))
    d["path"] = {0: "generic", 1: "tma", 2: "rows"}[d["path"]]
    return d
