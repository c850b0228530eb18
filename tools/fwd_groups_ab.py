#!/usr/bin/env python3
"""Plain fused forward on multi-sample launches (per-sample modulation), CUDA-event timed over
40 back-to-back launches: run once with AL_FWD_DYN_GROUPS=0 and once with 1 to A/B the chunked
multi-group tail.  Shapes B,S,D as arguments.  One JSON line per shape."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln._ops import fused_forward  # noqa: E402

dev = torch.device("cuda", 0)
for a in sys.argv[1:]:
    B, S, D = (int(v) for v in a.split(","))
    x = torch.randn(B, S, D, device=dev, dtype=torch.bfloat16)
    sc = 0.1 * torch.randn(B, D, device=dev, dtype=torch.bfloat16)
    sh = 0.1 * torch.randn(B, D, device=dev, dtype=torch.bfloat16)
    y = torch.empty_like(x)
    mu = torch.empty(B, S, device=dev)
    rs = torch.empty(B, S, device=dev)
    for _ in range(5):
        fused_forward(x, sc, sh, out=y, out_mean=mu, out_rstd=rs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(40):
        fused_forward(x, sc, sh, out=y, out_mean=mu, out_rstd=rs)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 40 * 1e3
    nb = 2 * B * S * D * 2 + 8 * B * S + 4 * B * D
    print(json.dumps({"dyn_groups": os.environ.get("AL_FWD_DYN_GROUPS", "1"), "shape": [B, S, D],
                      "us": round(us, 1), "GBps": round(nb / us / 1e3, 1)}), flush=True)
    del x, y
    torch.cuda.empty_cache()
