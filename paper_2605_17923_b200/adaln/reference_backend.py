"""The reference's internal backend protocol, served by the sm_100a kernels.

The reference picks a kernel module once at import (``_select_backend``,
/root/reference/pkg/src/adaptiveload/adaln/__init__.py:38-53) and calls four functions on it
with float64 numpy arrays:

    forward(x, scale, shift, eps) -> (y, mu, rstd)                   _kernels_numba.py:37-42
    backward_dx(dy, x, scale, mu, rstd) -> dx                         _kernels_numba.py:65-68
    backward_naive(dy, x, scale, mu, rstd) -> (dx, dscale, dshift)    _kernels_numba.py:86-91
    dtile_reduce(dy, x, mu, rstd, d_tile, n_tile, fp32_accum)         _kernels_numba.py:130-137
        -> (dscale, dshift)

This module implements exactly that protocol on the GPU (fp64 kernels, inputs copied to the
current CUDA device, results copied back), so the reference package can adopt it with a
one-line change in ``_select_backend``.  Validation stays in the reference's
own API layer, as it does for the numba/numpy backends.
"""

from __future__ import annotations

import numpy as np
import torch

from ._ops import fused_backward, fused_forward


def _dev(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(
        torch.device("cuda", torch.cuda.current_device()))


def forward(x, scale, shift, eps):
    y, mu, rstd = fused_forward(_dev(x), _dev(scale), _dev(shift), float(eps))
    return y.cpu().numpy(), mu.cpu().numpy(), rstd.cpu().numpy()


def backward_naive(dy, x, scale, mu, rstd):
    dx, dscale, dshift = fused_backward(_dev(dy), _dev(x), _dev(scale), _dev(mu), _dev(rstd),
                                        deterministic=True)
    return dx.cpu().numpy(), dscale.cpu().numpy(), dshift.cpu().numpy()


def backward_dx(dy, x, scale, mu, rstd):
    return backward_naive(dy, x, scale, mu, rstd)[0]


def dtile_reduce(dy, x, mu, rstd, d_tile, n_tile, fp32_accum):
    """dscale/dshift with the reference TileConfig (n_tile bounds the per-CTA partial height).

    dscale/dshift do not depend on scale; the fused kernel also forms dx, which is dropped.
    fp32_accum: the GPU accumulates fp64 inputs in fp64 (the stricter contract).
    """
    del fp32_accum
    x = np.ascontiguousarray(x, dtype=np.float64)
    zero_scale = np.zeros(x.shape[1])
    _, dscale, dshift = fused_backward(_dev(dy), _dev(x), _dev(zero_scale), _dev(mu), _dev(rstd),
                                       d_tile=int(d_tile), n_tile=int(n_tile), deterministic=True)
    return dscale.cpu().numpy(), dshift.cpu().numpy()
