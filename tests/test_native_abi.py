"""CPU checks of the C-ABI boundary: the library loads and exports exactly what the header declares."""

import re
from pathlib import Path

import pytest

from paper_2605_17923_b200 import _native as nat
from paper_2605_17923_b200 import _build

HEADER = Path(__file__).resolve().parent.parent / "include" / "adaln_b200.h"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"AL_API\s+[\w\s\*]+?\b(al_\w+)\s*\(", text)))


def test_header_declares_the_abi():
    syms = header_symbols()
    assert {"al_adaln_forward", "al_adaln_backward", "al_adaln_backward_workspace_bytes",
            "al_abi_version", "al_last_error"} <= set(syms)


def test_library_exports_every_header_symbol():
    lib = nat.load()
    for s in header_symbols():
        assert hasattr(lib, s), s
    assert sorted(nat.exported_symbols()) == header_symbols()


def test_library_is_sm100a():
    log = (_build.LIBDIR / "ptxas.log").read_text()
    assert "for 'sm_100a'" in log
    assert "adaln_fwd_rows" in log and "adaln_fwd_wide" in log and "adaln_bwd_tma" in log and "adaln_bwd_reduce" in log


def test_abi_version_and_errors_without_gpu():
    lib = nat.load()
    assert lib.al_abi_version() == nat.ABI_VERSION
    # argument validation happens before any CUDA call
    assert lib.al_set_tuning(2, 0, 0, 0, 0, 0) == nat.AL_ERR_VALUE
    assert "kernel" in nat.last_error()
    assert lib.al_set_tuning(0, 3, 0, 0, 0, 0) == nat.AL_ERR_VALUE
    assert lib.al_adaln_forward(None, None, None, None, None, None, 1, 4, 0, 0, nat.AL_F32,
                                1e-6, None, None) == nat.AL_ERR_SHAPE
    assert lib.al_adaln_forward(None, None, None, None, None, None, 1, 4, 8, 0, 9, 1e-6, None,
                                None) == nat.AL_ERR_DTYPE
    assert lib.al_adaln_forward(None, None, None, None, None, None, 1, 4, 8, 0, nat.AL_F32,
                                0.0, None, None) == nat.AL_ERR_VALUE
    # empty problems are no-ops
    assert lib.al_adaln_forward(None, None, None, None, None, None, 0, 4, 8, 0, nat.AL_F32,
                                1e-6, None, None) == nat.AL_OK
    # tile bounds use the reference's InvalidTile rule
    rc = lib.al_adaln_backward(None, None, None, None, None, None, None, None, None, 0,
                               1, 4, 8, 0, nat.AL_F32, 9, 1, 0, None, None)
    assert rc == nat.AL_ERR_TILE


def test_check_maps_status_codes():
    from paper_2605_17923_b200.errors import InvalidTile, NativeLibraryError, ShapeMismatch

    with pytest.raises(ShapeMismatch):
        nat.check(nat.AL_ERR_SHAPE, "x")
    with pytest.raises(InvalidTile):
        nat.check(nat.AL_ERR_TILE, "x")
    with pytest.raises(ValueError):
        nat.check(nat.AL_ERR_VALUE, "x")
    with pytest.raises(NativeLibraryError):
        nat.check(nat.AL_ERR_CUDA, "x")
