"""Fused gated residual + AdaLN forward (al_adaln_gate_residual_forward), SURVEY.md 8(f) #4.

The oracle is the reference's forward (oracle.forward_batched, restating _kernels_numba.py:18-42)
applied to x_out = x + gate * f computed in fp64 and rounded to the storage dtype, exactly the
composition the reference's block performs with two calls.  Tolerances as the rest of the suite:
fp32 1e-5, bf16 2e-2 relative (max|a-r| / max|r|), fp64 1e-11.
"""

import numpy as np
import pytest
import torch

import oracle
from conftest import max_rel_err
from paper_2605_17923_b200 import _native as nat
from paper_2605_17923_b200.adaln import gate_residual_adaln
from paper_2605_17923_b200.adaln._ops import (fused_backward, fused_forward,
                                              fused_gate_residual_backward,
                                              fused_gate_residual_forward)
from paper_2605_17923_b200.errors import NonFiniteInput, ShapeMismatch

pytestmark = pytest.mark.gpu

TOL = {torch.float64: 1e-11, torch.float32: 1e-5, torch.bfloat16: 2e-2, torch.float16: 5e-3}


def f64(t):
    return t.detach().double().cpu().numpy()


def make(b, s, d, dtype, device, seed=0, per_sample=True):
    g = torch.Generator(device="cpu").manual_seed(seed)
    mshape = (b, d) if per_sample else (d,)
    x = torch.randn(b, s, d, generator=g).to(dtype).to(device)
    f = torch.randn(b, s, d, generator=g).to(dtype).to(device)
    gate = (0.5 * torch.randn(*mshape, generator=g)).to(dtype).to(device)
    sc = (0.1 * torch.randn(*mshape, generator=g)).to(dtype).to(device)
    sh = (0.1 * torch.randn(*mshape, generator=g)).to(dtype).to(device)
    return x, f, gate, sc, sh


def oracle_gate_residual(x, f, gate, sc, sh, eps=1e-6):
    """x_out in fp64 rounded to x's dtype, then the reference forward on it."""
    gb = gate[:, None, :] if gate.dim() == 2 else gate
    xo = (x.double() + gb.double() * f.double()).to(x.dtype)
    b, s, d = x.shape
    scb = sc if sc.dim() == 2 else sc.expand(b, d)
    shb = sh if sh.dim() == 2 else sh.expand(b, d)
    y, mu, rs = oracle.forward_batched(f64(xo), f64(scb), f64(shb), eps, threads=0)
    return f64(xo), y, mu, rs


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16, torch.float64])
@pytest.mark.parametrize("shape", [(2, 97, 256), (2, 33, 1536), (1, 300, 5120), (1, 5, 8),
                                   (3, 7, 12288), (2, 17, 3)])
def test_matches_oracle(dtype, shape, cuda):
    b, s, d = shape
    x, f, gate, sc, sh = make(b, s, d, dtype, cuda, seed=b + s + d)
    xo, y, mu, rs = fused_gate_residual_forward(x, f, gate, sc, sh)
    xoo, yo, muo, rso = oracle_gate_residual(x, f, gate, sc, sh)
    tol = TOL[dtype]
    assert max_rel_err(f64(xo), xoo) <= tol
    if d > 1:
        assert max_rel_err(f64(y), yo) <= tol
        assert max_rel_err(f64(mu).ravel(), muo.ravel()) <= max(tol, 1e-5)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("shape", [(2, 300, 1536), (1, 200, 5120), (2, 9, 12288)])
def test_y_equals_forward_of_x_out_bitwise(dtype, shape, cuda):
    """The fused kernel's y/mean/rstd are exactly the one-row-per-warp forward applied to its
    x_out -- the mixed-precision 16-bit kernel (variant 4) for 16-bit rows of <= 8 vectors per
    lane, the packed rows kernel (variant 1) otherwise; rows too wide for either take the
    unfused composition (residual kernel, then the default forward)."""
    b, s, d = shape
    x, f, gate, sc, sh = make(b, s, d, dtype, cuda, seed=7)
    xo, y, mu, rs = fused_gate_residual_forward(x, f, gate, sc, sh)
    nvec = d * x.element_size() // 16
    rows_kernel = nvec <= 32 * 24
    variant = 4 if (x.element_size() == 2 and nvec <= 32 * 8) else 1
    try:
        nat.set_tuning(0, variant=variant if rows_kernel else 0)
        y2, mu2, rs2 = fused_forward(xo, sc, sh)
    finally:
        nat.set_tuning(0)
    assert torch.equal(y, y2) and torch.equal(mu, mu2) and torch.equal(rs, rs2)


def test_x_out_single_rounding(cuda):
    """x_out = round(fma(gate, f, x)) in fp32: at most half an ulp of bf16 from the fp64 value."""
    x, f, gate, sc, sh = make(2, 64, 1536, torch.bfloat16, cuda, seed=3)
    xo, *_ = fused_gate_residual_forward(x, f, gate, sc, sh)
    exact = (x.double() + gate.double()[:, None, :] * f.double())
    mism = (xo != exact.to(torch.bfloat16)).float().mean().item()
    assert mism < 1e-3  # only ties of the double rounding fp64->fp32->bf16 may differ


def test_broadcast_gate_and_2d(cuda):
    x, f, gate, sc, sh = make(3, 40, 512, torch.float32, cuda, seed=5, per_sample=False)
    xo, y, mu, rs = fused_gate_residual_forward(x, f, gate, sc, sh)
    xoo, yo, _, _ = oracle_gate_residual(x, f, gate, sc, sh)
    assert max_rel_err(f64(y), yo) <= 1e-5
    xo2, y2, _, _ = fused_gate_residual_forward(x.view(-1, 512), f.view(-1, 512), gate, sc, sh)
    assert torch.equal(y2.view_as(y), y) and torch.equal(xo2.view_as(xo), xo)


def test_misaligned_takes_unfused_path(cuda):
    base = torch.randn(2 * 33 * 256 + 1, device=cuda)
    x = base[1:].view(2, 33, 256)
    _, f, gate, sc, sh = make(2, 33, 256, torch.float32, cuda, seed=9)
    xo, y, _, _ = fused_gate_residual_forward(x, f, gate, sc, sh)
    xoo, yo, _, _ = oracle_gate_residual(x, f, gate, sc, sh)
    assert max_rel_err(f64(xo), xoo) <= 1e-6
    assert max_rel_err(f64(y), yo) <= 1e-5


def test_errors(cuda):
    x, f, gate, sc, sh = make(2, 8, 64, torch.float32, cuda)
    with pytest.raises(ShapeMismatch):
        fused_gate_residual_forward(x, f[:, :4], gate, sc, sh)
    with pytest.raises(ShapeMismatch):
        fused_gate_residual_forward(x, f, gate[0], sc, sh)
    with pytest.raises(ValueError):
        fused_gate_residual_forward(x, f, gate, sc, sh, eps=0.0)
    f2 = f.clone()
    f2[1, 3, 5] = float("nan")
    with pytest.raises(NonFiniteInput):
        fused_gate_residual_forward(x, f2, gate, sc, sh, check_finite=True)
    g2 = gate.clone()
    g2[0, 1] = float("inf")
    with pytest.raises(NonFiniteInput):
        fused_gate_residual_forward(x, f, g2, sc, sh, check_finite=True)
    lib = nat.load()
    p = x.data_ptr()
    rc = lib.al_adaln_gate_residual_forward(p, f.data_ptr(), gate.data_ptr(), sc.data_ptr(),
                                            sh.data_ptr(), p, p, p, p, 2, 8, 64, 64,
                                            nat.AL_F32, 1e-6, None, None)
    assert rc == nat.AL_ERR_VALUE  # x_out aliases x


def test_empty(cuda):
    x, f, gate, sc, sh = make(2, 0, 64, torch.bfloat16, cuda)
    xo, y, mu, rs = fused_gate_residual_forward(x, f, gate, sc, sh)
    assert xo.shape == x.shape and y.numel() == 0


def torch_block(x, f, gate, sc, sh, eps):
    xo = x + gate[:, None, :] * f
    mu = xo.mean(-1, keepdim=True)
    var = xo.var(-1, unbiased=False, keepdim=True)
    y = (xo - mu) / torch.sqrt(var + eps) * (1 + sc[:, None, :]) + sh[:, None, :]
    return xo, y


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_autograd_matches_torch_fp32(dtype, cuda):
    b, s, d = 2, 129, 1536
    x, f, gate, sc, sh = make(b, s, d, dtype, cuda, seed=21)
    g = torch.Generator(device="cpu").manual_seed(22)
    gxo = torch.randn(b, s, d, generator=g).to(dtype).to(cuda)
    gy = torch.randn(b, s, d, generator=g).to(dtype).to(cuda)
    ins = [t.clone().requires_grad_(True) for t in (x, f, gate, sc, sh)]
    xo, y = gate_residual_adaln(*ins, 1e-6)
    torch.autograd.backward([xo, y], [gxo, gy])
    ref = [t.detach().float().clone().requires_grad_(True) for t in (x, f, gate, sc, sh)]
    xr, yr = torch_block(*ref, 1e-6)
    torch.autograd.backward([xr, yr], [gxo.float(), gy.float()])
    tol = 1e-5 if dtype == torch.float32 else 2e-2
    assert max_rel_err(f64(y), f64(yr)) <= tol
    assert max_rel_err(f64(xo), f64(xr)) <= tol
    for a, r in zip(ins, ref):
        assert a.grad.dtype == a.dtype
        assert max_rel_err(f64(a.grad), f64(r.grad)) <= (1e-4 if dtype == torch.float32 else 2e-2)


def test_autograd_only_y_used(cuda):
    """x_out unused downstream: its gradient is zero and the node still runs."""
    x, f, gate, sc, sh = make(1, 64, 512, torch.float32, cuda, seed=2)
    ins = [t.clone().requires_grad_(True) for t in (x, f, gate, sc, sh)]
    _, y = gate_residual_adaln(*ins)
    y.sum().backward()
    ref = [t.detach().clone().requires_grad_(True) for t in (x, f, gate, sc, sh)]
    _, yr = torch_block(*ref, 1e-6)
    yr.sum().backward()
    for a, r in zip(ins, ref):
        assert max_rel_err(f64(a.grad), f64(r.grad)) <= 1e-4


def test_composed_backward_uses_fused_kernel(cuda):
    """dx of the node = fused_backward at x_out + the residual gradient."""
    x, f, gate, sc, sh = make(1, 100, 1024, torch.bfloat16, cuda, seed=4)
    xo, y, mu, rs = fused_gate_residual_forward(x, f, gate, sc, sh)
    gy = torch.randn_like(y)
    dxn, _, _ = fused_backward(gy, xo, sc, mu, rs)
    ins = [t.clone().requires_grad_(True) for t in (x, f, gate, sc, sh)]
    _, y2 = gate_residual_adaln(*ins)
    y2.backward(gy)
    assert torch.equal(ins[0].grad, dxn)


def test_graph_capture(cuda):
    x, f, gate, sc, sh = make(2, 256, 1536, torch.bfloat16, cuda, seed=6)
    nat.ensure_device(cuda.index)
    ref = fused_gate_residual_forward(x, f, gate, sc, sh)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fused_gate_residual_forward(x, f, gate, sc, sh)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = fused_gate_residual_forward(x, f, gate, sc, sh)
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(out, ref):
        assert torch.equal(a, b)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float64])
@pytest.mark.parametrize("shape,per_sample", [((2, 97, 256), True), ((3, 300, 1536), True),
                                              ((1, 200, 5120), True), ((4, 33, 512), False),
                                              ((2, 40, 8192), True)])
def test_residual_backward_kernel_vs_float64(dtype, shape, per_sample, cuda):
    """al_gate_residual_backward: dx = dxn + gxo, df = gate * dx, dgate = sum_s f * dx."""
    b, s, d = shape
    if d * torch.tensor([], dtype=dtype).element_size() > 2048 * 16:
        pytest.skip("wider than the kernel's 2048 16-byte vectors per row")
    _, f, gate, _, _ = make(b, s, d, dtype, cuda, seed=s + d, per_sample=per_sample)
    g = torch.Generator(device="cpu").manual_seed(5)
    dxn = torch.randn(b, s, d, generator=g).to(dtype).to(cuda)
    gxo = torch.randn(b, s, d, generator=g).to(dtype).to(cuda)
    dx, df, dgate = fused_gate_residual_backward(dxn, gxo, f, gate)
    G = (dxn.double() + gxo.double()).to(dtype).double()  # dx is stored rounded, then drives df/dgate
    gb = gate.double()[:, None, :] if per_sample else gate.double()
    tol = TOL[dtype]
    assert max_rel_err(f64(dx), f64(G)) <= tol
    assert max_rel_err(f64(df), f64(G * gb)) <= tol
    ref = (f.double() * G).sum(dim=1 if per_sample else (0, 1))
    assert max_rel_err(f64(dgate), f64(ref)) <= (1e-11 if dtype == torch.float64 else 1e-5)
    again = fused_gate_residual_backward(dxn, gxo, f, gate)
    assert all(torch.equal(a, c) for a, c in zip((dx, df, dgate), again))
    dx2, _, dgate2 = fused_gate_residual_backward(dxn, None, f, gate)  # no upstream residual grad
    assert torch.equal(dx2, dxn)
    assert max_rel_err(f64(dgate2), f64((f.double() * dxn.double()).sum(dim=1 if per_sample else (0, 1)))) <= (
        1e-11 if dtype == torch.float64 else 1e-5)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16, torch.float64])
@pytest.mark.parametrize("shape,per_sample", [((2, 97, 1000), True), ((1, 64, 13), False),
                                              ((3, 50, 3), True), ((2, 40, 40000), True)])
def test_residual_backward_generic_kernel(dtype, shape, per_sample, cuda):
    """Widths that are not 16-byte rows (and wider than the vector kernel) take the generic
    kernel: same arithmetic, checked against the float64 restatement; no torch fallback."""
    b, s, d = shape
    _, f, gate, _, _ = make(b, s, d, dtype, cuda, seed=s + d, per_sample=per_sample)
    g = torch.Generator(device="cpu").manual_seed(7)
    dxn = torch.randn(b, s, d, generator=g).to(dtype).to(cuda)
    gxo = torch.randn(b, s, d, generator=g).to(dtype).to(cuda)
    dx, df, dgate = fused_gate_residual_backward(dxn, gxo, f, gate)
    G = (dxn.double() + gxo.double()).to(dtype).double()
    gb = gate.double()[:, None, :] if per_sample else gate.double()
    tol = TOL[dtype]
    assert max_rel_err(f64(dx), f64(G)) <= tol
    assert max_rel_err(f64(df), f64(G * gb)) <= tol
    ref = (f.double() * G).sum(dim=1 if per_sample else (0, 1))
    assert max_rel_err(f64(dgate), f64(ref)) <= (1e-11 if dtype == torch.float64 else 1e-5)


def test_residual_backward_generic_equals_vector_kernel(cuda):
    """A misaligned view forces the generic kernel on a shape the vector kernel also takes: the
    outputs are bit-identical."""
    b, s, d = 2, 300, 1536
    _, f, gate, _, _ = make(b, s, d, torch.bfloat16, cuda, seed=11)
    g = torch.Generator(device="cpu").manual_seed(12)
    dxn = torch.randn(b, s, d, generator=g).to(torch.bfloat16).to(cuda)
    gxo = torch.randn(b, s, d, generator=g).to(torch.bfloat16).to(cuda)
    ref = fused_gate_residual_backward(dxn, gxo, f, gate)
    buf = torch.empty(b * s * d + 1, dtype=torch.bfloat16, device=cuda)
    mis = buf[1:].view(b, s, d)  # 2-byte offset: not 16-byte aligned
    mis.copy_(dxn)
    out = fused_gate_residual_backward(mis, gxo, f, gate)
    for a, r in zip(out, ref):
        assert torch.equal(a, r)
