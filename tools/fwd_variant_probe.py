#!/usr/bin/env python3
"""Forward GB/s per rows-kernel variant (al_set_tuning variant) at given shapes, bf16:
    python tools/fwd_variant_probe.py B S D [variants...]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import fused_forward  # noqa: E402

B, S, D = (int(a) for a in sys.argv[1:4])
variants = [int(a) for a in sys.argv[4:]] or [0, 4, 6]
dev = torch.device("cuda", 0)
x = torch.randn(B, S, D, device=dev).to(torch.bfloat16)
sc = (0.1 * torch.randn(B, D, device=dev)).to(torch.bfloat16)
sh = (0.1 * torch.randn(B, D, device=dev)).to(torch.bfloat16)
nb = 2 * x.numel() * 2 + 8 * B * S + 4 * B * D
for v in variants:
    nat.set_tuning(0, variant=v)
    for _ in range(5):
        fused_forward(x, sc, sh)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        fused_forward(x, sc, sh)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 50
    print(json.dumps({"B": B, "S": S, "D": D, "variant": v, "ms": round(ms, 4),
                      "gbs": round(nb / ms / 1e6, 1),
                      "plan": nat.describe_launch(0, B, S, D, D, nat.AL_BF16)}), flush=True)
nat.set_tuning(0)
