"""Autograd node for the fused operator: the "single atomic node" of PAPER.md.

Saves exactly what ``activation_bytes(..., MemoryMode.FUSED)`` accounts for -- the input x and
the per-row (mean, rstd) -- plus the [B, D] scale vector.  Backward runs the fused kernel pair
(dx + two-stage dscale/dshift reduction); no intermediate N x D tensor is ever materialised.
"""

from __future__ import annotations

import torch

from ._ops import (fused_backward, fused_forward, fused_gate_residual_backward,
                   fused_gate_residual_forward, fused_qk_rmsnorm_backward,
                   fused_qk_rmsnorm_forward)


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


class FusedGateResidualAdaLN(torch.autograd.Function):
    """(x_out, y) = (x + gate * f, AdaLN(x + gate * f)) as one node (al_adaln_gate_residual_forward).

    Saves x_out, f, gate, scale and the row statistics.  Backward, with upstream (g_xo, g_y):
        dxn, dscale, dshift = fused AdaLN backward of g_y at x_out      (K2 + K3)
        G = g_xo + dxn;  dx = G;  df = gate * G;  dgate = sum_s f * G   (one kernel + K3)
    """

    @staticmethod
    def forward(ctx, x, f, gate, scale, shift, eps: float = 1e-6):
        x_out, y, mean, rstd = fused_gate_residual_forward(x, f, gate, scale, shift, eps)
        ctx.save_for_backward(x_out, f, gate, scale, mean, rstd)
        ctx.mod_dtypes = (gate.dtype, scale.dtype, shift.dtype)
        return x_out, y

    @staticmethod
    def backward(ctx, g_xo, g_y):
        x_out, f, gate, scale, mean, rstd = ctx.saved_tensors
        # autograd materialises an unused output's gradient as zeros, so both are tensors here
        dxn, dsc, dsh = fused_backward(g_y, x_out, scale, mean, rstd)
        # one pass: G = dxn + g_xo, df = gate * G, dgate = sum_s f * G (the vector kernel for
        # 16-byte rows, the generic kernel -- same arithmetic -- for any other width/alignment)
        G, df, dgate = fused_gate_residual_backward(dxn, g_xo.to(dxn.dtype), f, gate)
        return (G, df, dgate.to(ctx.mod_dtypes[0]), dsc.to(ctx.mod_dtypes[1]),
                dsh.to(ctx.mod_dtypes[2]), None)


def gate_residual_adaln(x: torch.Tensor, f: torch.Tensor, gate: torch.Tensor, scale: torch.Tensor,
                        shift: torch.Tensor, eps: float = 1e-6):
    """(x + gate * f, LN(x + gate * f) * (1 + scale) + shift), fused forward, composed backward."""
    return FusedGateResidualAdaLN.apply(x, f, gate, scale, shift, eps)


class FusedQKRMSNorm(torch.autograd.Function):
    """(q_n, k_n, v) from a packed [..., 3D] projection: full-width RMSNorm of q and k with
    weights wq, wk (Wan-2.1's norm_q / norm_k), v passed through contiguous.  One forward and one
    backward kernel (plus the deterministic dw reduction); the backward writes d(qkv) whole."""

    @staticmethod
    def forward(ctx, qkv, wq, wk, eps: float = 1e-6):
        qn, kn, v, rstd = fused_qk_rmsnorm_forward(qkv, wq, wk, eps, copy_v=True)
        ctx.save_for_backward(qkv, wq, wk, rstd)
        ctx.w_dtypes = (wq.dtype, wk.dtype)
        return qn, kn, v

    @staticmethod
    def backward(ctx, dqn, dkn, dv):
        qkv, wq, wk, rstd = ctx.saved_tensors
        dqkv, dwq, dwk = fused_qk_rmsnorm_backward(qkv, wq, wk, rstd, dqn, dkn, dv)
        return dqkv, dwq.to(ctx.w_dtypes[0]), dwk.to(ctx.w_dtypes[1]), None


def qk_rmsnorm(qkv: torch.Tensor, wq: torch.Tensor, wk: torch.Tensor, eps: float = 1e-6):
    """(RMSNorm(q) * wq, RMSNorm(k) * wk, v) of a packed [..., 3D] qkv projection, fused."""
    return FusedQKRMSNorm.apply(qkv, wq, wk, eps)
