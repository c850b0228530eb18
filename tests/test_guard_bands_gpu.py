"""Out-of-bounds evidence without compute-sanitizer (closed on this GPU pool): every output is
carved out of a larger buffer whose guard bands before and after hold a canary bit pattern,
and every input sits between NaN guard bands.  After the call the canaries must be intact (no
write outside an output) and the outputs finite and equal to a run on plain tensors (no read
outside an input feeding a result).  Ragged shapes and every kernel path of the ABI."""

import pytest
import torch

from paper_2605_17923_b200 import _native as nat
from paper_2605_17923_b200.adaln._ops import (backward_workspace_bytes, fused_backward,
                                              fused_forward, fused_gate_residual_backward,
                                              fused_gate_residual_forward,
                                              fused_qk_rmsnorm_backward, fused_qk_rmsnorm_forward)

pytestmark = pytest.mark.gpu

GUARD = 4096  # elements on each side


def guarded(shape, dtype, device, fill=None):
    """(view, whole buffer) with the view in the middle of canary/NaN guard bands."""
    n = 1
    for s in shape:
        n *= s
    buf = torch.empty(n + 2 * GUARD, dtype=dtype, device=device)
    if dtype in (torch.float32, torch.float64, torch.bfloat16, torch.float16):
        buf.fill_(float("nan"))
    else:
        buf.fill_(0x5A)
    v = buf[GUARD:GUARD + n].view(*shape)
    if fill is not None:
        v.copy_(fill)
    return v, buf


def canary_ok(buf, n):
    head, tail = buf[:GUARD], buf[GUARD + n:]
    if buf.dtype.is_floating_point:
        return bool(torch.isnan(head).all() and torch.isnan(tail).all())
    return bool((head == 0x5A).all() and (tail == 0x5A).all())


CASES = [(2, 37, 1024, torch.bfloat16), (1, 129, 1536, torch.float32), (3, 9, 12288, torch.bfloat16),
         (2, 17, 5120, torch.bfloat16), (2, 5, 24, torch.float32), (1, 33, 2048, torch.float64),
         (1, 12001, 256, torch.bfloat16), (1, 20000, 512, torch.float16)]


@pytest.mark.parametrize("b,s,d,dt", CASES)
@pytest.mark.parametrize("det", [False, True])
def test_adaln_fwd_bwd_guard_bands(b, s, d, dt, det, cuda):
    g = torch.Generator(device="cpu").manual_seed(b * s + d)
    x0 = torch.randn(b, s, d, generator=g).to(dt).to(cuda)
    dy0 = torch.randn(b, s, d, generator=g).to(dt).to(cuda)
    sc0 = (0.1 * torch.randn(b, d, generator=g)).to(dt).to(cuda)
    sh0 = (0.1 * torch.randn(b, d, generator=g)).to(dt).to(cuda)
    ref_f = fused_forward(x0, sc0, sh0)
    ref_b = fused_backward(dy0, x0, sc0, ref_f[1], ref_f[2], deterministic=True)

    x, _ = guarded((b, s, d), dt, cuda, x0)
    dy, _ = guarded((b, s, d), dt, cuda, dy0)
    sc, _ = guarded((b, d), dt, cuda, sc0)
    sh, _ = guarded((b, d), dt, cuda, sh0)
    sdt = torch.float64 if dt == torch.float64 else torch.float32
    y, yb = guarded((b, s, d), dt, cuda)
    mu, mub = guarded((b, s), sdt, cuda)
    rs, rsb = guarded((b, s), sdt, cuda)
    fused_forward(x, sc, sh, out=y, out_mean=mu, out_rstd=rs)
    dx, dxb = guarded((b, s, d), dt, cuda)
    dsc, dscb = guarded((b, d), sdt, cuda)
    dsh, dshb = guarded((b, d), sdt, cuda)
    nws = backward_workspace_bytes(x, sc)
    ws, wsb = guarded((nws,), torch.uint8, cuda)
    ws.zero_()
    fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=det)
    torch.cuda.synchronize()
    for buf, n in ((yb, b * s * d), (mub, b * s), (rsb, b * s), (dxb, b * s * d),
                   (dscb, b * d), (dshb, b * d), (wsb, nws)):
        assert canary_ok(buf, n)
    assert torch.equal(y, ref_f[0]) and torch.equal(rs, ref_f[2])
    assert torch.equal(dx, ref_b[0])
    assert torch.isfinite(dsc).all() and torch.isfinite(dsh).all()
    if det:
        assert torch.equal(dsc, ref_b[1]) and torch.equal(dsh, ref_b[2])


@pytest.mark.parametrize("b,s,d,dt", [(2, 37, 1024, torch.bfloat16), (2, 10, 1000, torch.bfloat16),
                                      (1, 300, 5120, torch.float32), (3, 7, 40, torch.float64)])
def test_gate_residual_guard_bands(b, s, d, dt, cuda):
    g = torch.Generator(device="cpu").manual_seed(d)
    x0 = torch.randn(b, s, d, generator=g).to(dt).to(cuda)
    f0 = torch.randn(b, s, d, generator=g).to(dt).to(cuda)
    gate0 = (0.1 * torch.randn(b, d, generator=g)).to(dt).to(cuda)
    ref = fused_gate_residual_forward(x0, f0, gate0, gate0, gate0)
    refb = fused_gate_residual_backward(x0, f0, f0, gate0)
    x, _ = guarded((b, s, d), dt, cuda, x0)
    f, _ = guarded((b, s, d), dt, cuda, f0)
    gate, _ = guarded((b, d), dt, cuda, gate0)
    out = fused_gate_residual_forward(x, f, gate, gate, gate)
    outb = fused_gate_residual_backward(x, f, f, gate)
    torch.cuda.synchronize()
    for a, r in zip(out + outb, ref + refb):
        assert torch.equal(a, r)


def test_qk_rmsnorm_guard_bands(cuda):
    b, s, d = 2, 129, 1536
    g = torch.Generator(device="cpu").manual_seed(3)
    q0 = torch.randn(b, s, 3 * d, generator=g).to(torch.bfloat16).to(cuda)
    w0 = (1 + 0.1 * torch.randn(d, generator=g)).to(torch.bfloat16).to(cuda)
    ref = fused_qk_rmsnorm_forward(q0, w0, w0)
    qkv, _ = guarded((b, s, 3 * d), torch.bfloat16, cuda, q0)
    w, _ = guarded((d,), torch.bfloat16, cuda, w0)
    out = fused_qk_rmsnorm_forward(qkv, w, w)
    dq = torch.randn_like(out[0])
    refb = fused_qk_rmsnorm_backward(q0, w0, w0, ref[3], dq, dq, ref[2])
    outb = fused_qk_rmsnorm_backward(qkv, w, w, out[3], dq, dq, out[2])
    torch.cuda.synchronize()
    for a, r in zip(out, ref):
        assert torch.equal(a, r)
    for a, r in zip(outb, refb):
        assert torch.equal(a, r)
