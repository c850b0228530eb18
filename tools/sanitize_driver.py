#!/usr/bin/env python3
"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck): every kernel
path once -- rows forward (bf16, fp32), wide forward, generic forward/backward, TMA backward
with separate and fused stage 2, multi-sample groups, ragged tails."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

dev = torch.device("cuda", 0)
cases = [(2, 37, 1024, torch.bfloat16), (1, 129, 1536, torch.float32), (3, 9, 12288, torch.bfloat16),
         (2, 17, 5120, torch.bfloat16), (2, 5, 3, torch.float32), (1, 33, 2048, torch.float64)]
for b, s, d, dt in cases:
    x = torch.randn(b, s, d, device=dev).to(dt)
    dy = torch.randn_like(x)
    sc = (0.1 * torch.randn(b, d, device=dev)).to(dt)
    sh = (0.1 * torch.randn(b, d, device=dev)).to(dt)
    for fwd_variant in (0, 2, 5):
        nat.set_tuning(0, variant=fwd_variant)
        y, mu, rs = fused_forward(x, sc, sh, check_finite=True)
    nat.set_tuning(0)
    for bwd_variant in (0, 2):
        nat.set_tuning(1, variant=bwd_variant)
        fused_backward(dy, x, sc, mu, rs, check_finite=True)
    nat.set_tuning(1)
torch.cuda.synchronize()
print("sanitize driver ok")
