#!/usr/bin/env python3
"""Backward kernels side by side, eager launches timed by their own device timestamps:
default (work stealing), round-1 (tuning variant 4: dynamic tail / static when deterministic),
skewed pipeline (variant 3, R = 2).  Shapes: cfg2, cfg3 lengths, multi-sample batches.

    python tools/bwd_variants.py [iters]
"""
import json
import statistics as stt
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import (backward_workspace_bytes, fused_backward,  # noqa: E402
                                              fused_forward)

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
dev = torch.device("cuda", 0)
D = 5120
ts = torch.empty(iters, 2, dtype=torch.int64, device=dev)


def med_ts(fn):
    for _ in range(3):
        fn()
    ts[:, 0] = -1
    ts[:, 1] = 0
    torch.cuda.synchronize()
    nat.set_timestamps(ts.data_ptr(), iters)
    for _ in range(iters):
        fn()
    torch.cuda.synchronize()
    nat.set_timestamps(None)
    return stt.median([(e - b) / 1e3 for b, e in ts.cpu().tolist()])


for B, S in [(1, 1560), (1, 3600), (1, 7800), (1, 14040), (4, 1560), (8, 1560), (2, 7800),
             (1, 32760), (1, 75600)]:
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(B, S, D, device=dev, generator=g).to(torch.bfloat16)
    dy = torch.randn(B, S, D, device=dev, generator=g).to(torch.bfloat16)
    sc = (0.1 * torch.randn(B, D, device=dev, generator=g)).to(torch.bfloat16)
    _, mu, rs = fused_forward(x, sc, sc)
    bb = 3 * B * S * D * 2 + B * D * 2 + 8 * B * S + 8 * B * D
    out = (torch.empty_like(x), torch.empty(B, D, device=dev), torch.empty(B, D, device=dev))
    ws = torch.empty(backward_workspace_bytes(x, sc), dtype=torch.uint8, device=dev)
    res = {"B": B, "S": S}
    for name, var, R, det in (("default", 0, 0, True), ("r1_dyn", 4, 0, False), ("r1_det", 4, 0, True),
                              ("pipe_dyn", 3, 2, False), ("pipe_det", 3, 2, True)):
        nat.set_tuning(1, 0, R, 0, False, var)
        us = med_ts(lambda: fused_backward(dy, x, sc, mu, rs, out=out, workspace=ws, deterministic=det))
        res[name] = [round(us, 2), round(bb / us / 1e3, 1)]
    nat.set_tuning(1, 0, 0, 0, False, 0)
    print(json.dumps(res), flush=True)
    del x, dy, mu, rs, out, ws
