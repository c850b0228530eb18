#!/usr/bin/env python3
"""ncu driver (round 2): after warm-up, one launch each of the cfg2 forward (rows16, two-pass),
the cfg2 backward (dynamic tail and deterministic interleaved), and an S = 3 600 backward
(skewed pipeline)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

dev = torch.device("cuda", 0)
D = 5120
big = [torch.randn(1, 32760, D, device=dev).to(torch.bfloat16) for _ in range(2)]
small = [torch.randn(1, 3600, D, device=dev).to(torch.bfloat16) for _ in range(2)]
sc = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
for _ in range(2):
    y, mu, rs = fused_forward(big[0], sc, sc)
    fused_backward(big[1], big[0], sc, mu, rs, deterministic=False)
    fused_backward(big[1], big[0], sc, mu, rs, deterministic=True)
    y2, mu2, rs2 = fused_forward(small[0], sc, sc)
    fused_backward(small[1], small[0], sc, mu2, rs2)
torch.cuda.synchronize()
print("ok")
