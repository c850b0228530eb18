"""Fused Q/K RMSNorm of a packed QKV projection (al_qk_rmsnorm_forward / _backward).

The reference has no implementation of this op (it is named only in its design notes,
PAPER.md:301), so the checker is a float64 torch restatement of Wan-2.1's RMSNorm on the q and k
slices, with autograd for the gradients.  Tolerances as the rest of the suite: fp32 1e-5,
bf16 2e-2, fp16 5e-3 relative (max|a-r| / max|r|), fp64 1e-11.
"""

import pytest
import torch

from conftest import max_rel_err
from paper_2605_17923_b200 import _native as nat
from paper_2605_17923_b200.adaln import qk_rmsnorm
from paper_2605_17923_b200.adaln._ops import (fused_qk_rmsnorm_backward,
                                              fused_qk_rmsnorm_forward)
from paper_2605_17923_b200.errors import NativeLibraryError, ShapeMismatch

pytestmark = pytest.mark.gpu

TOL = {torch.float64: 1e-11, torch.float32: 1e-5, torch.bfloat16: 2e-2, torch.float16: 5e-3}


def f64(t):
    return t.detach().double().cpu().numpy()


def make(lead, d, dtype, device, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    qkv = torch.randn(*lead, 3 * d, generator=g).to(dtype).to(device)
    wq = (1 + 0.2 * torch.randn(d, generator=g)).to(dtype).to(device)
    wk = (1 + 0.2 * torch.randn(d, generator=g)).to(dtype).to(device)
    return qkv, wq, wk


def reference(qkv, wq, wk, eps=1e-6):
    d = qkv.shape[-1] // 3
    q, k, v = qkv.split(d, dim=-1)

    def rms(x, w):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w

    return rms(q, wq), rms(k, wk), v


SHAPES = [((2, 64), 256), ((1, 300), 1536), ((3, 33), 2048), ((2, 17), 1024), ((5,), 64)]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16, torch.float64])
@pytest.mark.parametrize("lead,d", SHAPES)
def test_forward_backward_vs_float64(dtype, lead, d, cuda):
    if d * torch.tensor([], dtype=dtype).element_size() > 4096:
        pytest.skip("wider than the kernel's 4 KB row slice")
    qkv, wq, wk = make(lead, d, dtype, cuda, seed=d)
    g = torch.Generator(device="cpu").manual_seed(d + 1)
    dqn, dkn, dv = (torch.randn(*lead, d, generator=g).to(dtype).to(cuda) for _ in range(3))
    qn, kn, vc, rstd = fused_qk_rmsnorm_forward(qkv, wq, wk)
    ref_in = [t.detach().double().requires_grad_(True) for t in (qkv, wq, wk)]
    rq, rk, rv = reference(*ref_in)
    tol = TOL[dtype]
    assert max_rel_err(f64(qn), f64(rq)) <= tol
    assert max_rel_err(f64(kn), f64(rk)) <= tol
    assert torch.equal(vc, qkv[..., 2 * d:])
    dqkv, dwq, dwk = fused_qk_rmsnorm_backward(qkv, wq, wk, rstd, dqn, dkn, dv)
    torch.autograd.backward([rq, rk, rv], [dqn.double(), dkn.double(), dv.double()])
    assert max_rel_err(f64(dqkv), f64(ref_in[0].grad)) <= tol
    red_tol = 1e-11 if dtype == torch.float64 else 1e-5
    assert max_rel_err(f64(dwq), f64(ref_in[1].grad)) <= max(red_tol, tol if dtype != torch.float32 else 1e-5)
    assert max_rel_err(f64(dwk), f64(ref_in[2].grad)) <= max(red_tol, tol if dtype != torch.float32 else 1e-5)


def test_deterministic_and_dv_optional(cuda):
    qkv, wq, wk = make((4, 500), 1536, torch.bfloat16, cuda, seed=3)
    dqn, dkn = torch.randn_like(qkv[..., :1536]), torch.randn_like(qkv[..., :1536])
    _, _, _, rstd = fused_qk_rmsnorm_forward(qkv, wq, wk)
    a = fused_qk_rmsnorm_backward(qkv, wq, wk, rstd, dqn, dkn)
    b = fused_qk_rmsnorm_backward(qkv, wq, wk, rstd, dqn, dkn)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    assert torch.count_nonzero(a[0][..., 2 * 1536:]) == 0  # dv slice untouched (zeros)
    qn, kn, vc, _ = fused_qk_rmsnorm_forward(qkv, wq, wk, copy_v=False)
    assert vc is None


def test_autograd_node_and_unused_outputs(cuda):
    qkv, wq, wk = make((2, 129), 1024, torch.float32, cuda, seed=9)
    ins = [t.clone().requires_grad_(True) for t in (qkv, wq, wk)]
    qn, kn, v = qk_rmsnorm(*ins)
    (qn.square().sum() + 0.5 * v.sum()).backward()  # kn unused: zero gradient flows
    ref = [t.detach().double().requires_grad_(True) for t in (qkv, wq, wk)]
    rq, rk, rv = reference(*ref)
    (rq.square().sum() + 0.5 * rv.sum()).backward()
    assert ref[2].grad is None and float(ins[2].grad.abs().max()) == 0.0  # wk: k_n unused
    for a, r in zip(ins[:2], ref[:2]):
        assert a.grad.dtype == a.dtype
        assert max_rel_err(f64(a.grad), f64(r.grad)) <= 1e-5


def test_errors_and_empty(cuda):
    qkv, wq, wk = make((2, 8), 4096, torch.bfloat16, cuda)
    with pytest.raises(ShapeMismatch):  # 8 KB rows: wider than the kernel takes
        fused_qk_rmsnorm_forward(qkv, wq, wk)
    qkv, wq, wk = make((2, 8), 256, torch.float32, cuda)
    with pytest.raises(ShapeMismatch):
        fused_qk_rmsnorm_forward(qkv[..., :-1], wq, wk)
    with pytest.raises(ShapeMismatch):
        fused_qk_rmsnorm_forward(qkv, wq[:-1], wk)
    with pytest.raises(ValueError):
        fused_qk_rmsnorm_forward(qkv, wq, wk, eps=0.0)
    lib = nat.load()
    rc = lib.al_qk_rmsnorm_forward(qkv.data_ptr(), 2 * 256, wq.data_ptr(), wk.data_ptr(),
                                   qkv.data_ptr(), qkv.data_ptr(), qkv.data_ptr(), qkv.data_ptr(),
                                   16, 256, nat.AL_F32, 1e-6, None, None)
    assert rc == nat.AL_ERR_SHAPE  # a v copy needs row_stride >= 3 * dim
    empty, wq0, wk0 = make((0,), 256, torch.float32, cuda)
    qn, kn, vc, rstd = fused_qk_rmsnorm_forward(empty, wq0, wk0)
    assert qn.shape == (0, 256)
    dqkv, dwq, dwk = fused_qk_rmsnorm_backward(empty, wq0, wk0, rstd, qn, kn, vc)
    assert dqkv.shape == (0, 768) and float(dwq.abs().sum()) == 0.0
    assert NativeLibraryError is not None


def test_graph_capture(cuda):
    qkv, wq, wk = make((2, 256), 1536, torch.bfloat16, cuda, seed=6)
    nat.ensure_device(cuda.index)
    ref = fused_qk_rmsnorm_forward(qkv, wq, wk)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fused_qk_rmsnorm_forward(qkv, wq, wk)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = fused_qk_rmsnorm_forward(qkv, wq, wk)
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(out, ref):
        assert torch.equal(a, b)
