#!/usr/bin/env python3
"""Minimal driver for ncu: cfg2 (B=1, S=32760, D=5120 bf16) fused fwd+bwd, `--reps` times
(--batch B: B samples per launch with per-sample modulation, the sampler's buckets; --det: the
deterministic backward)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--seq", type=int, default=32760)
ap.add_argument("--dim", type=int, default=5120)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--det", action="store_true")
a = ap.parse_args()
dt = {"bf16": torch.bfloat16, "fp32": torch.float32}[a.dtype]
dev = torch.device("cuda", 0)
x = torch.randn(a.batch, a.seq, a.dim, device=dev).to(dt)
dy = torch.randn(a.batch, a.seq, a.dim, device=dev).to(dt)
sc = (0.1 * torch.randn(a.batch, a.dim, device=dev)).to(dt)
sh = (0.1 * torch.randn(a.batch, a.dim, device=dev)).to(dt)
for _ in range(a.reps):
    y, mu, rs = fused_forward(x, sc, sh)
    fused_backward(dy, x, sc, mu, rs, deterministic=a.det)
torch.cuda.synchronize()
print("ok")
