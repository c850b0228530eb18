"""Autograd node for the fused operator: the "single atomic node" of PAPER.md.

Saves exactly what ``activation_bytes(..., MemoryMode.FUSED)`` accounts for -- the input x and
the per-row (mean, rstd) -- plus the [B, D] scale vector.  Backward runs the fused kernel pair
(dx + two-stage dscale/dshift reduction); no intermediate N x D tensor is ever materialised.
"""

from __future__ import annotations

import torch

from ._ops import fused_backward, fused_forward


class FusedAdaLNModulate(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, scale, shift, eps: float = 1e-6):
        y, mean, rstd = fused_forward(x, scale, shift, eps)
        ctx.save_for_backward(x, scale, mean, rstd)
        ctx.mod_dtypes = (scale.dtype, shift.dtype)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, scale, mean, rstd = ctx.saved_tensors
        dx, dscale, dshift = fused_backward(dy, x, scale, mean, rstd)
        return dx, dscale.to(ctx.mod_dtypes[0]), dshift.to(ctx.mod_dtypes[1]), None


def adaln_modulate(x: torch.Tensor, scale: torch.Tensor, shift: torch.Tensor,
                   eps: float = 1e-6) -> torch.Tensor:
    """y = LN(x) * (1 + scale) + shift with per-sample scale/shift [B, D] broadcast over S."""
    return FusedAdaLNModulate.apply(x, scale, shift, eps)
