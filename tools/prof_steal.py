#!/usr/bin/env python3
"""cfg2 driver for an ncu capture of the work-stealing backward (2 warm-ups, then 1 launch)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

S, D = 32760, 5120
dev = torch.device("cuda", 0)
x = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
dy = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
sc = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
y, mu, rs = fused_forward(x, sc, sc)
for _ in range(3):
    fused_backward(dy, x, sc, mu, rs)
torch.cuda.synchronize()
print("ok")
