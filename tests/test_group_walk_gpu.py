"""Group-sequential interleaved backward walk (adaln_bwd_tma with interleave = 2): deterministic
multi-sample launches of long samples (> 16 384 rows each) walk every sample like a
single-sample launch, one after the other, with G partial slots per sample (stage 2 slot map
tail0 = -2).  Checked: the oracle per sample, bit-identity run to run and inside a CUDA graph,
dx bit-identical to the non-deterministic schedule (same per-row arithmetic) and dscale/dshift
equal to it to fp32 summation order, and the fallback when the caller's workspace is the
pre-group-walk size (work stealing) giving the same results to fp32 order."""

import os

import numpy as np
import pytest
import torch

import oracle
from conftest import max_rel_err
from paper_2605_17923_b200 import _native as nat
from paper_2605_17923_b200.adaln._ops import backward_workspace_bytes, fused_backward, fused_forward

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(os.environ.get("AL_BWD_GROUP_WALK") == "0",
                                 reason="group walk disabled by AL_BWD_GROUP_WALK=0")]


def f64(t):
    return t.detach().double().cpu().numpy()


def _data(b, s, d, dtype, dev, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randn(b, s, d, generator=g).to(dtype).to(dev)
    dy = torch.randn(b, s, d, generator=g).to(dtype).to(dev)
    sc = (0.1 * torch.randn(b, d, generator=g)).to(dtype).to(dev)
    return x, dy, sc


SHAPES = [(2, 20000, 2048, torch.bfloat16), (3, 17001, 1024, torch.float32),
          (2, 16500, 1536, torch.float16), (2, 18000, 5120, torch.bfloat16)]


@pytest.mark.parametrize("b,s,d,dt", SHAPES)
def test_group_walk_vs_oracle_and_reproducible(b, s, d, dt, cuda):
    x, dy, sc = _data(b, s, d, dt, cuda, seed=s + d)
    _, mu, rs = fused_forward(x, sc, sc)
    first = fused_backward(dy, x, sc, mu, rs, deterministic=True)
    for _ in range(2):
        again = fused_backward(dy, x, sc, mu, rs, deterministic=True)
        for u, v in zip(first, again):
            assert torch.equal(u, v)
    # the non-deterministic schedule of the same launch: dx bit-identical (same per-row math),
    # dscale/dshift to fp32 summation order
    nd = fused_backward(dy, x, sc, mu, rs, deterministic=False)
    assert torch.equal(first[0], nd[0])
    assert max_rel_err(f64(first[1]), f64(nd[1])) <= 2e-6
    assert max_rel_err(f64(first[2]), f64(nd[2])) <= 2e-6
    # oracle, every sample's dscale / dshift, sampled dx rows
    h = lambda t: t.double().cpu().numpy()  # noqa: E731
    rows = np.random.default_rng(0).choice(s, 64, replace=False)
    for bi in range(b):
        dxo, dsco, dsho = oracle.backward_naive(h(dy[bi]), h(x[bi]), h(sc[bi]), h(mu[bi]),
                                                h(rs[bi]), threads=8)
        assert max_rel_err(f64(first[1][bi]), dsco) <= 1e-5
        assert max_rel_err(f64(first[2][bi]), dsho) <= 1e-5
        bar = 1e-5 if dt == torch.float32 else 2e-2
        assert max_rel_err(f64(first[0][bi])[rows], dxo[rows]) <= bar


def test_group_walk_fallback_with_pre_group_walk_workspace(cuda):
    """A C-ABI caller whose workspace is sized as before the group walk existed (static +
    stealing slots only) still gets a correct launch: it falls back to work stealing, same
    results to fp32 order (the Python layer always sizes by al_adaln_backward_workspace_bytes)."""
    b, s, d = 5, 17000, 1024
    x, dy, sc = _data(b, s, d, torch.bfloat16, cuda, seed=3)
    _, mu, rs = fused_forward(x, sc, sc)
    ref = fused_backward(dy, x, sc, mu, rs, deterministic=True)
    G = nat.describe_launch(1, b, s, d, d, nat.AL_BF16)["grid"]
    small = 2 * (G + b - 1 + 2 * G) * d * 4 + 16
    assert small < backward_workspace_bytes(x, sc)
    ws = torch.empty(small, dtype=torch.uint8, device=cuda)
    dx = torch.empty_like(x)
    dsc = torch.empty(b, d, device=cuda)
    dsh = torch.empty(b, d, device=cuda)
    rc = nat.load().al_adaln_backward(
        dy.data_ptr(), x.data_ptr(), sc.data_ptr(), mu.data_ptr(), rs.data_ptr(), dx.data_ptr(),
        dsc.data_ptr(), dsh.data_ptr(), ws.data_ptr(), small, b, s, d, d, nat.AL_BF16, 0, 0,
        nat.AL_BWD_DETERMINISTIC, None, torch.cuda.current_stream().cuda_stream)
    nat.check(rc, "al_adaln_backward")
    torch.cuda.synchronize()
    assert torch.equal(dx, ref[0])
    assert max_rel_err(f64(dsc), f64(ref[1])) <= 2e-6
    assert max_rel_err(f64(dsh), f64(ref[2])) <= 2e-6


def test_group_walk_in_cuda_graph(cuda):
    b, s, d = 2, 20000, 2048
    x, dy, sc = _data(b, s, d, torch.bfloat16, cuda, seed=9)
    _, mu, rs = fused_forward(x, sc, sc)
    ref = fused_backward(dy, x, sc, mu, rs, deterministic=True)
    dx = torch.empty_like(x)
    dsc = torch.empty(b, d, device=cuda)
    dsh = torch.empty(b, d, device=cuda)
    ws = torch.empty(backward_workspace_bytes(x, sc), dtype=torch.uint8, device=cuda)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=True)
        with torch.cuda.graph(g, stream=side):
            fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=True)
    torch.cuda.synchronize()
    for _ in range(3):
        dx.zero_()
        dsc.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(dx, ref[0])
        assert torch.equal(dsc, ref[1])
        assert torch.equal(dsh, ref[2])
