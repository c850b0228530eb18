"""Ring-slot reuse race guard for the backward (adaln_bwd_tma / adaln_bwd_steal): a deterministic
launch repeated many times must give bit-identical dx and dscale every time.  A consumer that
released its ring slot before the values it loaded from it had been consumed let the producer's
next TMA copy overwrite them: at 5 x 17 000 x 1 024 bf16 that corrupted 25 of 300 launches
(tools/bwd_race_stress.py) -- this catches that class of bug in a few hundred launches."""

import pytest
import torch

from paper_2605_17923_b200.adaln._ops import backward_workspace_bytes, fused_backward, fused_forward

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("b,s,d", [(5, 17000, 1024), (1, 20000, 1024), (3, 7001, 5120)])
def test_repeated_deterministic_backward_is_bit_identical(b, s, d, cuda):
    g = torch.Generator(device="cpu").manual_seed(b * s + d)
    x = torch.randn(b, s, d, generator=g).to(torch.bfloat16).to(cuda)
    dy = torch.randn(b, s, d, generator=g).to(torch.bfloat16).to(cuda)
    sc = (0.1 * torch.randn(b, d, generator=g)).to(torch.bfloat16).to(cuda)
    _, mu, rs = fused_forward(x, sc, sc)
    ref = [t.clone() for t in fused_backward(dy, x, sc, mu, rs, deterministic=True)]
    dx = torch.empty_like(x)
    dsc = torch.empty(b, d, device=cuda)
    dsh = torch.empty(b, d, device=cuda)
    ws = torch.empty(backward_workspace_bytes(x, sc), dtype=torch.uint8, device=cuda)
    bad = 0
    for _ in range(150):
        fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=True)
        bad += int(not (torch.equal(dx, ref[0]) and torch.equal(dsc, ref[1])))
    assert bad == 0, f"{bad} of 150 launches differ"
