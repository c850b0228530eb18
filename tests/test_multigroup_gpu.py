"""Multi-sample launches (the sampler's buckets: B samples of one length in one launch).

* forward: the dynamic row tail spans modulation groups (rows of a group other than the CTA's
  staged one read (1 + scale, shift) from global memory) -- every row must equal the same row
  computed by a one-sample launch, bit for bit, whichever path it took;
* backward stage 2 over many groups (adaln_bwd_reduce_grp, >= 8 groups without a dynamic tail)
  -- dscale/dshift vs the oracle-style fp64 reference, and per-sample equality with one-sample
  launches where the partial layout makes the sums identical;
* non-finite modulation rows in tail groups are still rejected.
"""

import pytest
import torch

from paper_2605_17923_b200.adaln import adaln_forward
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward
from paper_2605_17923_b200.errors import NonFiniteInput

pytestmark = pytest.mark.gpu


def _inputs(b, s, d, dt, cuda, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = (torch.randn(b, s, d, generator=g) * 2 + 0.5).to(dt).to(cuda)
    dy = torch.randn(b, s, d, generator=g).to(dt).to(cuda)
    sc = (0.3 * torch.randn(b, d, generator=g)).to(dt).to(cuda)
    sh = (0.3 * torch.randn(b, d, generator=g)).to(dt).to(cuda)
    return x, dy, sc, sh


# (40, 250, 5120): 10 000 rows, 8 000 in the tail across ~32 groups; (64, 160, 1536): the
# two-rows-per-warp width; (24, 999, 2048): ragged groups
@pytest.mark.parametrize("b,s,d,dt", [(40, 250, 5120, torch.bfloat16), (64, 160, 1536, torch.bfloat16),
                                      (24, 999, 2048, torch.float16), (30, 333, 5120, torch.float16)])
def test_forward_multigroup_tail_bitwise_per_sample(b, s, d, dt, cuda):
    x, _, sc, sh = _inputs(b, s, d, dt, cuda)
    y, mu, rs = fused_forward(x, sc, sh)
    for i in range(b):
        yi, mi, ri = fused_forward(x[i:i + 1], sc[i:i + 1], sh[i:i + 1])
        assert torch.equal(y[i:i + 1], yi), i
        assert torch.equal(mu[i:i + 1], mi) and torch.equal(rs[i:i + 1], ri), i
    # and against an fp32 torch restatement (the output rounding of 16-bit y)
    xf = x.float()
    ref = (xf - xf.mean(-1, keepdim=True)) / torch.sqrt(xf.var(-1, unbiased=False, keepdim=True) + 1e-6)
    ref = ref * (1 + sc.float()[:, None]) + sh.float()[:, None]
    assert (y.float() - ref).abs().max().item() <= 2e-2 * max(1.0, ref.abs().max().item())


@pytest.mark.parametrize("b,s,d,dt", [(40, 250, 5120, torch.bfloat16), (17, 96, 1024, torch.float32),
                                      (64, 33, 512, torch.float64), (20, 700, 2048, torch.bfloat16)])
@pytest.mark.parametrize("det", [False, True])
def test_backward_many_groups(b, s, d, dt, det, cuda):
    x, dy, sc, sh = _inputs(b, s, d, dt, cuda, seed=1)
    y, mu, rs = fused_forward(x, sc, sh)
    dx, dsc, dsh = fused_backward(dy, x, sc, mu, rs, deterministic=det)
    # fp64 reference of the column sums from the same saved statistics
    xh = (x.double() - mu.double()[..., None]) * rs.double()[..., None]
    ref_sc = (dy.double() * xh).sum(1)
    ref_sh = dy.double().sum(1)
    tol = 1e-9 if dt == torch.float64 else 2e-5
    scale_ = ref_sh.abs().max().item() + 1.0
    assert (dsc.double() - ref_sc).abs().max().item() <= tol * (ref_sc.abs().max().item() + 1.0) * 10
    assert (dsh.double() - ref_sh).abs().max().item() <= tol * scale_ * 10
    # run to run: bit-identical (no dynamic tail in many-group launches)
    dx2, dsc2, dsh2 = fused_backward(dy, x, sc, mu, rs, deterministic=det)
    assert torch.equal(dx, dx2) and torch.equal(dsc, dsc2) and torch.equal(dsh, dsh2)


def test_forward_multigroup_nonfinite_tail_scale(cuda):
    x, _, sc, sh = _inputs(40, 250, 5120, torch.bfloat16, cuda)
    sc[37, 4000] = float("nan")  # a group deep in the dynamic tail
    with pytest.raises(NonFiniteInput):
        adaln_forward(x, sc, sh)
    sc[37, 4000] = 0.0
    sh[39, 5] = float("inf")
    with pytest.raises(NonFiniteInput):
        adaln_forward(x, sc, sh)


@pytest.mark.parametrize("b,s,d", [(40, 250, 1536), (24, 999, 2048)])
def test_gate_residual_multigroup_tail_bitwise_per_sample(b, s, d, cuda):
    """The gated-residual twin's chunked multi-group tail (restages gate, 1 + scale, shift per
    chunk): every sample equal to a one-sample launch, bit for bit."""
    from paper_2605_17923_b200.adaln._ops import fused_gate_residual_forward

    g = torch.Generator(device="cpu").manual_seed(3)
    x = torch.randn(b, s, d, generator=g).to(torch.bfloat16).to(cuda)
    f = torch.randn(b, s, d, generator=g).to(torch.bfloat16).to(cuda)
    gate, sc, sh = ((0.3 * torch.randn(b, d, generator=g)).to(torch.bfloat16).to(cuda)
                    for _ in range(3))
    full = fused_gate_residual_forward(x, f, gate, sc, sh)
    for i in range(b):
        one = fused_gate_residual_forward(x[i:i + 1], f[i:i + 1], gate[i:i + 1], sc[i:i + 1],
                                          sh[i:i + 1])
        for a, r in zip(full, one):
            assert torch.equal(a[i:i + 1], r), i
