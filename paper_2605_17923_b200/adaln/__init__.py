"""Fused LayerNorm-Modulate (AdaLN) operator -- the reference's public operator API on B200.

Drop-in for ``adaptiveload.adaln`` (/root/reference/pkg/src/adaptiveload/adaln/__init__.py):
same names, argument meaning, result dataclasses and exception types (``__all__`` mirrors
adaln/__init__.py:23-35).  Every numeric result comes from the sm_100a kernels of
``libadaln_b200.so``; there is no CPU fallback and no backend dispatch (``BACKEND`` is fixed).

Argument kinds:
  * torch CUDA tensors: computed in their own dtype (fp32/bf16/fp16 in fp32 arithmetic, fp64 in
    fp64), results stay on the device.  x may be [N, D] (reference) or [B, S, D] with per-sample
    scale/shift [B, D] (the north-star layout; dscale/dshift come back [B, D]).
  * torch CPU tensors: streamed through the GPU in row chunks with host->device copies,
    kernels and device->host copies overlapped on two streams (``_host.py``); results come
    back in pinned host memory in the input dtype.  The forward keeps its device copy of x
    for a following backward on the same (unmodified, by version counter) tensor
    (``release_resident()`` frees it; ``AL_HOST_RESIDENT=0`` disables).
  * numpy arrays / sequences: the reference's semantics -- cast to float64 (``_as_f64``,
    adaln/__init__.py:81-85), computed in fp64 on the GPU, returned as float64 numpy arrays.

Non-finite inputs raise NonFiniteInput like the reference; the scan is folded into the kernels
(a device flag) instead of a separate host pass.  For CUDA tensors that check costs one
device->host read; pass ``check_finite=False`` (or use ``fused_forward``/``fused_backward``
from ``._ops``) on a training hot path.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np
import torch

from ..errors import InvalidTile, ShapeMismatch, StaleStats
from ._host import host_backward, host_forward, release_resident  # noqa: F401
from ._ops import fused_backward, fused_forward, fused_gate_residual_forward, geometry, stat_dtype  # noqa: F401

__all__ = [
    "AdalnOutput",
    "AdalnGrads",
    "TileConfig",
    "MemoryMode",
    "BACKEND",
    "adaln_forward",
    "adaln_backward_naive",
    "adaln_backward_dtile",
    "activation_bytes",
    "gradcheck",
    "GradcheckReport",
]

# The reference picks "numba" or "numpy" at import (adaln/__init__.py:38-53); this build has one.
BACKEND = "cuda-sm100a"


@dataclass(frozen=True)
class AdalnOutput:
    y: object
    mu: object
    rstd: object


@dataclass(frozen=True)
class AdalnGrads:
    dx: object
    dscale: object
    dshift: object


@dataclass(frozen=True)
class TileConfig:
    """Reference tile hint (adaln/__init__.py:70-73).

    Validated with the reference bounds.  On the GPU, ``n_tile`` bounds the number of rows
    folded into one stage-1 (per-CTA) partial; ``d_tile`` is accepted for API parity -- column
    ownership is fixed by the kernel's 16-byte vectors (each thread owns its feature columns).
    """

    d_tile: int
    n_tile: int


class MemoryMode(enum.Enum):
    NAIVE = "naive"
    FUSED = "fused"


# --------------------------------------------------------------------------- argument staging
class _Staged:
    """Moves host arguments to the device and results back, per the kind of the inputs."""

    def __init__(self, *args):
        self.kind = None
        for a in args:
            if isinstance(a, torch.Tensor):
                k = "cuda" if a.is_cuda else "torch-cpu"
            else:
                k = "numpy"
            if self.kind is None:
                self.kind = k
            elif self.kind != k:
                # mixed kinds: follow the reference and treat everything as host float64
                self.kind = "numpy"
        if self.kind == "cuda":
            self.device = next(a.device for a in args if isinstance(a, torch.Tensor))
        else:
            self.device = torch.device("cuda", torch.cuda.current_device())

    def put(self, a, f64: bool = True):
        if self.kind == "cuda":
            return a
        if self.kind == "torch-cpu":
            return a.to(self.device, non_blocking=True)
        if isinstance(a, torch.Tensor):
            a = a.detach().cpu().numpy()
        arr = np.ascontiguousarray(np.asarray(a), dtype=np.float64)
        return torch.from_numpy(arr).to(self.device)

    def get(self, t: torch.Tensor):
        if self.kind == "cuda":
            return t
        if self.kind == "torch-cpu":
            return t.cpu()
        return t.cpu().numpy()


def adaln_forward(x, scale, shift, eps: float = 1e-6, *, check_finite: bool = True) -> AdalnOutput:
    """Normalize each token row and modulate: y = xhat * (1 + scale) + shift.

    Mirrors adaln/__init__.py:99-108 (errors: ShapeMismatch, NonFiniteInput, ValueError).
    """
    st = _Staged(x, scale, shift)
    if st.kind == "torch-cpu":  # host buffers: chunked H2D / compute / D2H pipeline
        geometry(x, scale, shift)
        if eps <= 0:
            raise ValueError("eps must be positive")
        y, mu, rstd = host_forward(x, scale.to(x.dtype), shift.to(x.dtype), eps, True, st.device)
        return AdalnOutput(y=y, mu=mu, rstd=rstd)
    xd, sc, sh = st.put(x), st.put(scale), st.put(shift)
    geometry(xd, sc, sh)  # ShapeMismatch before touching the GPU
    if eps <= 0:
        raise ValueError("eps must be positive")
    y, mu, rstd = fused_forward(xd, sc, sh, eps, check_finite=check_finite or st.kind != "cuda")
    return AdalnOutput(y=st.get(y), mu=st.get(mu), rstd=st.get(rstd))


def _check_cached(x: torch.Tensor, mu: torch.Tensor, rstd: torch.Tensor) -> None:
    """StaleStats when cached (mu, rstd) do not describe x (adaln/__init__.py:111-116)."""
    rows = x.shape[:-1]
    n = int(np.prod(rows)) if len(rows) else 1
    for t in (mu, rstd):
        if tuple(t.shape) not in (tuple(rows), (n,)):
            raise StaleStats(
                f"cached stats shapes {tuple(mu.shape)}/{tuple(rstd.shape)} do not match "
                f"rows {tuple(rows)}")


def _validate_backward(dy, x, scale, mu, rstd, d_tile: int, n_tile: int):
    if tuple(dy.shape) != tuple(x.shape):
        raise ShapeMismatch(f"dy shape {tuple(dy.shape)} != x shape {tuple(x.shape)}")
    g = geometry(x, scale)
    _check_cached(x, mu, rstd)
    if d_tile or n_tile:
        rows_per_group = g.seq if g.mod_stride else g.batch * g.seq
        if not (1 <= d_tile <= g.dim and 1 <= n_tile <= rows_per_group):
            raise InvalidTile(
                f"tile config {TileConfig(d_tile, n_tile)} out of bounds for "
                f"N={rows_per_group}, D={g.dim}")
    return g


def _backward(dy, x, scale, mu, rstd, d_tile: int, n_tile: int, check_finite: bool) -> AdalnGrads:
    st = _Staged(dy, x, scale, mu, rstd)
    if st.kind == "torch-cpu":  # host buffers: chunked H2D / compute / D2H pipeline
        _validate_backward(dy, x, scale, mu, rstd, d_tile, n_tile)
        dx, dscale, dshift = host_backward(dy.to(x.dtype), x, scale.to(x.dtype), mu, rstd,
                                           d_tile, n_tile, True, st.device)
        return AdalnGrads(dx=dx, dscale=dscale, dshift=dshift)
    dyd, xd, sc = st.put(dy), st.put(x), st.put(scale)
    mud, rsd = st.put(mu), st.put(rstd)
    g = _validate_backward(dyd, xd, sc, mud, rsd, d_tile, n_tile)
    sdt = stat_dtype(xd.dtype)
    mud = mud.reshape(g.stats_shape).to(sdt)
    rsd = rsd.reshape(g.stats_shape).to(sdt)
    # the reference API keeps the reference's fixed per-feature accumulation order
    dx, dscale, dshift = fused_backward(dyd, xd, sc, mud, rsd, d_tile=d_tile, n_tile=n_tile,
                                        check_finite=check_finite or st.kind != "cuda",
                                        deterministic=True)
    return AdalnGrads(dx=st.get(dx), dscale=st.get(dscale), dshift=st.get(dshift))


def adaln_backward_naive(dy, x, scale, mu, rstd, *, check_finite: bool = True) -> AdalnGrads:
    """Backward with the default reduction tiling (adaln/__init__.py:119-130)."""
    return _backward(dy, x, scale, mu, rstd, 0, 0, check_finite)


def adaln_backward_dtile(dy, x, scale, mu, rstd, tiles: TileConfig, fp32_accum: bool = False,
                         *, check_finite: bool = True) -> AdalnGrads:
    """Backward with an explicit tile configuration (adaln/__init__.py:133-158).

    dx is identical to the naive variant.  The GPU always accumulates stage-1 partials in the
    compute precision (fp32 for 16/32-bit inputs, fp64 for fp64 inputs) and sums partials across
    CTAs in fp64, so ``fp32_accum`` needs no separate path: the fp32-accumulation contract
    (<= 1e-5 relative, test_adaln.py:170-179) holds either way.
    """
    del fp32_accum
    return _backward(dy, x, scale, mu, rstd, int(tiles.d_tile), int(tiles.n_tile), check_finite)


def activation_bytes(n: int, d: int, element_bytes: int, stat_bytes: int, mode: MemoryMode) -> int:
    """Activation footprint model (adaln/__init__.py:161-175).

    NAIVE saves three N x D tensors (input, normalized, modulated intermediate) plus two per-row
    statistics; FUSED saves the input plus (mu, rstd) -- exactly what ``FusedAdaLNModulate``
    keeps for backward.
    """
    if min(n, d, element_bytes, stat_bytes) < 1:
        raise ValueError("all counts must be >= 1")
    saved_rows = 3 if mode is MemoryMode.NAIVE else 1
    return saved_rows * n * d * element_bytes + 2 * n * stat_bytes


from ._gradcheck import DEFAULT_SIZES, GradcheckReport, gradcheck  # noqa: E402
from .autograd import (FusedAdaLNModulate, FusedGateResidualAdaLN, FusedQKRMSNorm,  # noqa: E402,F401
                       adaln_modulate, gate_residual_adaln, qk_rmsnorm)
