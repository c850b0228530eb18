#!/usr/bin/env python3
"""Small cfg2 driver for ncu captures of the backward stage-1 kernels: 2 warm-up rounds, then one
fwd + one backward per variant (0 = adaln_bwd_tma, 3 = adaln_bwd_pipe R=2), dynamic tail.

    python tools/prof_bwd.py [variants...]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

variants = [int(v) for v in sys.argv[1:]] or [0, 3]
S, D = 32760, 5120
dev = torch.device("cuda", 0)
x = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
dy = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
sc = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
sh = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
for _ in range(2):
    for v in variants:
        nat.set_tuning(1, 0, 2 if v == 3 else 0, 0, False, v)
        y, mu, rs = fused_forward(x, sc, sh)
        fused_backward(dy, x, sc, mu, rs, deterministic=False)
torch.cuda.synchronize()
print("ok")
