"""Device-level entry points: torch CUDA tensors in, torch CUDA tensors out.

These are the thin host-side callers of the C ABI (``include/adaln_b200.h``).  Torch is only
plumbing here: it owns the device memory (caching allocator) and the current stream; all
arithmetic runs in the sm_100a kernels of ``libadaln_b200.so``.

Layouts accepted (the reference accepts only the first, adaln/__init__.py:88-96):
  * x [N, D] with scale/shift [D]            -> mean/rstd [N],    dscale/dshift [D]
  * x [B, S, D] with scale/shift [B, D]      -> mean/rstd [B, S], dscale/dshift [B, D]
  * x [B, S, D] with scale/shift [D]         -> mean/rstd [B, S], dscale/dshift [D]
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .. import _native as nat
from ..errors import NonFiniteInput, ShapeMismatch

_DTYPE_CODE = {
    torch.float32: nat.AL_F32,
    torch.bfloat16: nat.AL_BF16,
    torch.float16: nat.AL_F16,
    torch.float64: nat.AL_F64,
}


def dtype_code(dt: torch.dtype) -> int:
    try:
        return _DTYPE_CODE[dt]
    except KeyError:
        raise TypeError(f"unsupported dtype {dt}; expected float32/bfloat16/float16/float64") from None


def stat_dtype(dt: torch.dtype) -> torch.dtype:
    """mean/rstd/dscale/dshift dtype: fp64 for fp64 inputs, fp32 otherwise."""
    return torch.float64 if dt == torch.float64 else torch.float32


@dataclass(frozen=True)
class Geometry:
    batch: int
    seq: int
    dim: int
    mod_stride: int  # 0 = scale/shift broadcast over every row
    stats_shape: tuple
    grad_shape: tuple


def geometry(x: torch.Tensor, scale: torch.Tensor, shift: torch.Tensor | None = None) -> Geometry:
    if x.dim() == 2:
        n, d = x.shape
        b, s = 1, n
        stats_shape = (n,)
    elif x.dim() == 3:
        b, s, d = x.shape
        stats_shape = (b, s)
    else:
        raise ShapeMismatch(f"x must be 2-D [N, D] or 3-D [B, S, D], got {tuple(x.shape)}")
    mods = [scale] if shift is None else [scale, shift]
    shapes = [tuple(m.shape) for m in mods]
    if all(sh == (d,) for sh in shapes):
        return Geometry(b, s, d, 0, stats_shape, (d,))
    if x.dim() == 3 and all(sh == (b, d) for sh in shapes):
        return Geometry(b, s, d, d, stats_shape, (b, d))
    want = f"({d},)" if x.dim() == 2 else f"({d},) or ({b}, {d})"
    raise ShapeMismatch(f"scale/shift must have shape {want}, got {shapes}")


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class _NoGuard:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


_NO_GUARD = _NoGuard()


def _on(device: torch.device):
    """Make `device` current around a library call: the C ABI plans and launches on the CUDA
    current device (cudaGetDevice), and the stream it gets belongs to `device`.  A no-op when
    `device` is already current (the common case), so the guard costs one query per call."""
    if torch.cuda.current_device() == device.index:
        return _NO_GUARD
    return torch.cuda.device(device)


def _prep(t: torch.Tensor, dt: torch.dtype, device: torch.device) -> torch.Tensor:
    if t.device != device:
        raise ShapeMismatch(f"all tensors must be on {device}, got {t.device}")
    if t.dtype != dt:
        t = t.to(dt)
    return t.contiguous()


def _raise_if_flagged(flag: torch.Tensor | None, what: str) -> None:
    if flag is not None and int(flag.item()) != 0:
        raise NonFiniteInput(f"{what} contains NaN or Inf")


def _out_like(t: torch.Tensor | None, shape, dtype, dev, what: str) -> torch.Tensor:
    """A caller-supplied output (checked) or a fresh one."""
    if t is None:
        return torch.empty(shape, dtype=dtype, device=dev)
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype or t.device != dev or not t.is_contiguous():
        raise ShapeMismatch(f"{what}: expected contiguous {dtype} {tuple(shape)} on {dev}, "
                            f"got {t.dtype} {tuple(t.shape)} on {t.device}")
    return t


def fused_forward(x: torch.Tensor, scale: torch.Tensor, shift: torch.Tensor, eps: float = 1e-6,
                  *, check_finite: bool = False, out: torch.Tensor | None = None,
                  flag: torch.Tensor | None = None, out_mean: torch.Tensor | None = None,
                  out_rstd: torch.Tensor | None = None):
    """y, mean, rstd = AdaLN forward (one HBM pass).  Asynchronous unless check_finite.

    ``flag`` (device int32[1]): accumulate the non-finite flag there without synchronising
    (the caller checks it once, e.g. after a chunked host pipeline).  ``out`` / ``out_mean`` /
    ``out_rstd``: caller-owned outputs (e.g. buffers reused by every step of a captured graph)."""
    if not x.is_cuda:
        raise ShapeMismatch("fused_forward takes CUDA tensors; use adaln_forward for host data")
    if eps <= 0:
        raise ValueError("eps must be positive")
    g = geometry(x, scale, shift)
    dev = x.device
    nat.ensure_device(dev.index)
    x = _prep(x, x.dtype, dev)
    scale = _prep(scale, x.dtype, dev)
    shift = _prep(shift, x.dtype, dev)
    y = _out_like(out, x.shape, x.dtype, dev, "out")
    sdt = stat_dtype(x.dtype)
    mean = _out_like(out_mean, g.stats_shape, sdt, dev, "out_mean")
    rstd = _out_like(out_rstd, g.stats_shape, sdt, dev, "out_rstd")
    own_flag = check_finite and flag is None
    if own_flag:
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
    with _on(dev):
        rc = nat.load().al_adaln_forward(
            x.data_ptr(), scale.data_ptr(), shift.data_ptr(), y.data_ptr(), mean.data_ptr(),
            rstd.data_ptr(), g.batch, g.seq, g.dim, g.mod_stride, dtype_code(x.dtype), float(eps),
            flag.data_ptr() if flag is not None else None, _stream_ptr(dev))
    nat.check(rc, "al_adaln_forward")
    if own_flag:
        _raise_if_flagged(flag, "x/scale/shift")
    return y, mean, rstd


def fused_gate_residual_forward(x: torch.Tensor, f: torch.Tensor, gate: torch.Tensor,
                                scale: torch.Tensor, shift: torch.Tensor, eps: float = 1e-6, *,
                                check_finite: bool = False, flag: torch.Tensor | None = None):
    """x_out = x + gate * f;  y, mean, rstd = AdaLN(x_out)  -- one pass (al_adaln_gate_residual_forward).

    ``gate`` has the shape of scale/shift ([D] or [B, D]); returns (x_out, y, mean, rstd)."""
    if not x.is_cuda:
        raise ShapeMismatch("fused_gate_residual_forward takes CUDA tensors")
    if eps <= 0:
        raise ValueError("eps must be positive")
    g = geometry(x, scale, shift)
    geometry(x, gate)  # same broadcast rules as scale
    if tuple(gate.shape) != tuple(scale.shape):
        raise ShapeMismatch(f"gate shape {tuple(gate.shape)} != scale shape {tuple(scale.shape)}")
    if tuple(f.shape) != tuple(x.shape):
        raise ShapeMismatch(f"f shape {tuple(f.shape)} != x shape {tuple(x.shape)}")
    dev = x.device
    nat.ensure_device(dev.index)
    x = _prep(x, x.dtype, dev)
    f = _prep(f, x.dtype, dev)
    gate = _prep(gate, x.dtype, dev)
    scale = _prep(scale, x.dtype, dev)
    shift = _prep(shift, x.dtype, dev)
    x_out = torch.empty_like(x)
    y = torch.empty_like(x)
    sdt = stat_dtype(x.dtype)
    mean = torch.empty(g.stats_shape, dtype=sdt, device=dev)
    rstd = torch.empty(g.stats_shape, dtype=sdt, device=dev)
    own_flag = check_finite and flag is None
    if own_flag:
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
    with _on(dev):
        rc = nat.load().al_adaln_gate_residual_forward(
            x.data_ptr(), f.data_ptr(), gate.data_ptr(), scale.data_ptr(), shift.data_ptr(),
            x_out.data_ptr(), y.data_ptr(), mean.data_ptr(), rstd.data_ptr(), g.batch, g.seq, g.dim,
            g.mod_stride, dtype_code(x.dtype), float(eps),
            flag.data_ptr() if flag is not None else None, _stream_ptr(dev))
    nat.check(rc, "al_adaln_gate_residual_forward")
    if own_flag:
        _raise_if_flagged(flag, "x/f/gate/scale/shift")
    return x_out, y, mean, rstd


def backward_workspace_bytes(x: torch.Tensor, scale: torch.Tensor, n_tile: int = 0) -> int:
    """Bytes of scratch fused_backward needs for these shapes (al_adaln_backward_workspace_bytes)."""
    g = geometry(x, scale)
    with _on(x.device):
        n = nat.load().al_adaln_backward_workspace_bytes(g.batch, g.seq, g.dim, g.mod_stride,
                                                          dtype_code(x.dtype), n_tile)
    if n < 0:
        nat.check(nat.AL_ERR_SHAPE, "al_adaln_backward_workspace_bytes")
    return max(int(n), 16)


def fused_backward(dy: torch.Tensor, x: torch.Tensor, scale: torch.Tensor, mean: torch.Tensor,
                   rstd: torch.Tensor, *, d_tile: int = 0, n_tile: int = 0,
                   check_finite: bool = False, flag: torch.Tensor | None = None,
                   deterministic: bool | None = None, out: tuple | None = None,
                   workspace: torch.Tensor | None = None):
    """dx, dscale, dshift in one pass over (dy, x) + a fixed-order cross-CTA reduction.

    deterministic: True fixes the assignment of rows to partial sums (dscale/dshift
    bit-identical run to run, the reference's fixed per-feature order).  False hands a single
    sample's stages (or the last sample's, in a launch of more than 4 long samples) to whichever
    SM is free (~1 % faster at cfg2), which moves that sample's dscale/dshift at fp32 rounding
    level from run to run -- dx is identical either way.  None (default) follows
    ``torch.are_deterministic_algorithms_enabled()``.
    ``out`` = (dx, dscale, dshift) and ``workspace`` (uint8, at least
    ``al_adaln_backward_workspace_bytes``): caller-owned buffers, e.g. reused by a captured graph.
    """
    if deterministic is None:
        deterministic = torch.are_deterministic_algorithms_enabled()
    if not x.is_cuda:
        raise ShapeMismatch("fused_backward takes CUDA tensors; use adaln_backward_* for host data")
    g = geometry(x, scale)
    if tuple(dy.shape) != tuple(x.shape):
        raise ShapeMismatch(f"dy shape {tuple(dy.shape)} != x shape {tuple(x.shape)}")
    dev = x.device
    nat.ensure_device(dev.index)
    x = _prep(x, x.dtype, dev)
    dy = _prep(dy, x.dtype, dev)
    scale = _prep(scale, x.dtype, dev)
    sdt = stat_dtype(x.dtype)
    mean = _prep(mean, sdt, dev)
    rstd = _prep(rstd, sdt, dev)
    lib = nat.load()
    code = dtype_code(x.dtype)
    with _on(dev):
        ws_bytes = lib.al_adaln_backward_workspace_bytes(g.batch, g.seq, g.dim, g.mod_stride,
                                                         code, n_tile)
    if ws_bytes < 0:
        nat.check(nat.AL_ERR_SHAPE, "al_adaln_backward_workspace_bytes")
    if workspace is None:
        ws = torch.empty(max(int(ws_bytes), 16), dtype=torch.uint8, device=dev)
    else:
        if workspace.device != dev or workspace.dtype != torch.uint8 or workspace.numel() < ws_bytes:
            raise ShapeMismatch(f"workspace: need >= {ws_bytes} uint8 bytes on {dev}")
        ws = workspace
        ws_bytes = workspace.numel()
    o = out if out is not None else (None, None, None)
    dx = _out_like(o[0], x.shape, x.dtype, dev, "out[0] (dx)")
    dscale = _out_like(o[1], g.grad_shape, sdt, dev, "out[1] (dscale)")
    dshift = _out_like(o[2], g.grad_shape, sdt, dev, "out[2] (dshift)")
    own_flag = check_finite and flag is None
    if own_flag:
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
    with _on(dev):
        rc = lib.al_adaln_backward(
            dy.data_ptr(), x.data_ptr(), scale.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
            dx.data_ptr(), dscale.data_ptr(), dshift.data_ptr(), ws.data_ptr(), int(ws_bytes),
            g.batch, g.seq, g.dim, g.mod_stride, code, d_tile, n_tile,
            nat.AL_BWD_DETERMINISTIC if deterministic else 0,
            flag.data_ptr() if flag is not None else None, _stream_ptr(dev))
    nat.check(rc, "al_adaln_backward")
    if own_flag:
        _raise_if_flagged(flag, "dy/x/scale")
    return dx, dscale, dshift


# ------------------------------------------------------------------ fused Q/K RMSNorm
def fused_qk_rmsnorm_forward(qkv: torch.Tensor, wq: torch.Tensor, wk: torch.Tensor,
                             eps: float = 1e-6, *, copy_v: bool = True,
                             check_finite: bool = False):
    """q_n, k_n (, v) = RMSNorm over the full width of the q and k slices of a packed
    [..., 3D] projection (al_qk_rmsnorm_forward).  Returns (q_n, k_n, v or None, rstd[..., 2])."""
    if not qkv.is_cuda:
        raise ShapeMismatch("fused_qk_rmsnorm_forward takes CUDA tensors")
    if eps <= 0:
        raise ValueError("eps must be positive")
    if qkv.shape[-1] % 3:
        raise ShapeMismatch(f"last dim of qkv must be 3 * D, got {qkv.shape[-1]}")
    d = qkv.shape[-1] // 3
    if tuple(wq.shape) != (d,) or tuple(wk.shape) != (d,):
        raise ShapeMismatch(f"wq/wk must have shape ({d},), got {tuple(wq.shape)}, {tuple(wk.shape)}")
    dev = qkv.device
    nat.ensure_device(dev.index)
    qkv = _prep(qkv, qkv.dtype, dev)
    wq = _prep(wq, qkv.dtype, dev)
    wk = _prep(wk, qkv.dtype, dev)
    lead = qkv.shape[:-1]
    n = qkv.numel() // (3 * d) if qkv.numel() else 0
    qn = torch.empty(*lead, d, dtype=qkv.dtype, device=dev)
    kn = torch.empty_like(qn)
    vc = torch.empty_like(qn) if copy_v else None
    rstd = torch.empty(*lead, 2, dtype=stat_dtype(qkv.dtype), device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev) if check_finite else None
    with _on(dev):
        rc = nat.load().al_qk_rmsnorm_forward(
            qkv.data_ptr(), 3 * d, wq.data_ptr(), wk.data_ptr(), qn.data_ptr(), kn.data_ptr(),
            vc.data_ptr() if vc is not None else None, rstd.data_ptr(), n, d, dtype_code(qkv.dtype),
            float(eps), flag.data_ptr() if flag is not None else None, _stream_ptr(dev))
    nat.check(rc, "al_qk_rmsnorm_forward")
    _raise_if_flagged(flag, "qkv")
    return qn, kn, vc, rstd


def fused_qk_rmsnorm_backward(qkv: torch.Tensor, wq: torch.Tensor, wk: torch.Tensor,
                              rstd: torch.Tensor, dqn: torch.Tensor, dkn: torch.Tensor,
                              dv: torch.Tensor | None = None):
    """d(qkv) = [dq | dk | dv] and dwq, dwk (fp32; fp64 for fp64) -- al_qk_rmsnorm_backward."""
    d = qkv.shape[-1] // 3
    dev = qkv.device
    nat.ensure_device(dev.index)
    qkv = _prep(qkv, qkv.dtype, dev)
    wq = _prep(wq, qkv.dtype, dev)
    wk = _prep(wk, qkv.dtype, dev)
    sdt = stat_dtype(qkv.dtype)
    rstd = _prep(rstd, sdt, dev)
    dqn = _prep(dqn, qkv.dtype, dev)
    dkn = _prep(dkn, qkv.dtype, dev)
    if dv is not None:
        dv = _prep(dv, qkv.dtype, dev)
    n = qkv.numel() // (3 * d) if qkv.numel() else 0
    lib = nat.load()
    code = dtype_code(qkv.dtype)
    with _on(dev):
        ws_bytes = lib.al_qk_rmsnorm_backward_workspace_bytes(n, d, code)
    if ws_bytes < 0:
        nat.check(nat.AL_ERR_SHAPE, "al_qk_rmsnorm_backward_workspace_bytes")
    ws = torch.empty(max(int(ws_bytes), 16), dtype=torch.uint8, device=dev)
    dqkv = torch.empty_like(qkv) if dv is not None else torch.zeros_like(qkv)
    dwq = torch.empty(d, dtype=sdt, device=dev)
    dwk = torch.empty(d, dtype=sdt, device=dev)
    with _on(dev):
        rc = lib.al_qk_rmsnorm_backward(
            qkv.data_ptr(), 3 * d, wq.data_ptr(), wk.data_ptr(), rstd.data_ptr(), dqn.data_ptr(),
            dkn.data_ptr(), dv.data_ptr() if dv is not None else None, dqkv.data_ptr(),
            dwq.data_ptr(), dwk.data_ptr(), ws.data_ptr(), int(ws_bytes), n, d, code, None,
            _stream_ptr(dev))
    nat.check(rc, "al_qk_rmsnorm_backward")
    return dqkv, dwq, dwk


def fused_gate_residual_backward(dxn: torch.Tensor, gxo: torch.Tensor | None, f: torch.Tensor,
                                 gate: torch.Tensor):
    """dx = dxn + gxo, df = gate * dx, dgate = sum_s f * dx in one pass
    (al_gate_residual_backward).  gate: [D] or [B, D]; dgate is fp32 (fp64 for fp64)."""
    g = geometry(dxn, gate)
    dev = dxn.device
    nat.ensure_device(dev.index)
    dt = dxn.dtype
    dxn = _prep(dxn, dt, dev)
    f = _prep(f, dt, dev)
    gate = _prep(gate, dt, dev)
    if gxo is not None:
        gxo = _prep(gxo, dt, dev)
    lib = nat.load()
    code = dtype_code(dt)
    with _on(dev):
        ws_bytes = lib.al_gate_residual_backward_workspace_bytes(g.batch, g.seq, g.dim,
                                                                 g.mod_stride, code)
    if ws_bytes < 0:
        nat.check(nat.AL_ERR_SHAPE, "al_gate_residual_backward_workspace_bytes")
    ws = torch.empty(max(int(ws_bytes), 16), dtype=torch.uint8, device=dev)
    dx = torch.empty_like(dxn)
    df = torch.empty_like(dxn)
    dgate = torch.empty(g.grad_shape, dtype=stat_dtype(dt), device=dev)
    with _on(dev):
        rc = lib.al_gate_residual_backward(
            dxn.data_ptr(), gxo.data_ptr() if gxo is not None else None, f.data_ptr(),
            gate.data_ptr(), dx.data_ptr(), df.data_ptr(), dgate.data_ptr(), ws.data_ptr(),
            int(ws_bytes), g.batch, g.seq, g.dim, g.mod_stride, code, _stream_ptr(dev))
    nat.check(rc, "al_gate_residual_backward")
    return dx, df, dgate
