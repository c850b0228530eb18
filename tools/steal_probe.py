#!/usr/bin/env python3
"""Backward stage-1 balancing schemes at cfg2 and a few lengths, eager launches timed by the
kernels' own device timestamps (no graph capture: each capture would take a protocol slot).
Prints median us of `iters` launches for the default (work stealing) and the round-1 scheme.

    AL_STEAL_CHUNK=16 python tools/steal_probe.py [iters] [tag]
"""
import json
import os
import statistics as stt
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import (backward_workspace_bytes, fused_backward,  # noqa: E402
                                              fused_forward)

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
tag = sys.argv[2] if len(sys.argv) > 2 else "steal"
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


for B, S in [(1, 32760), (1, 75600), (4, 1560), (1, 7800), (1, 3600)]:
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(B, S, D, device=dev, generator=g).to(torch.bfloat16)
    dy = torch.randn(B, S, D, device=dev, generator=g).to(torch.bfloat16)
    sc = (0.1 * torch.randn(B, D, device=dev, generator=g)).to(torch.bfloat16)
    _, mu, rs = fused_forward(x, sc, sc)
    bb = 3 * B * S * D * 2 + B * D * 2 + 8 * B * S + 8 * B * D
    out = (torch.empty_like(x), torch.empty(B, D, device=dev), torch.empty(B, D, device=dev))
    ws = torch.empty(backward_workspace_bytes(x, sc), dtype=torch.uint8, device=dev)
    res = {"tag": tag, "B": B, "S": S, "chunk": os.environ.get("AL_STEAL_CHUNK", "8"),
           "pool": os.environ.get("AL_STEAL_POOL", "2")}
    c0 = nat.steal_count(0)
    res["steal_us"] = round(med_ts(lambda: fused_backward(dy, x, sc, mu, rs, out=out, workspace=ws)), 2)
    res["stolen_per_launch"] = round((nat.steal_count(0) - c0) / (iters + 3), 1)
    nat.set_tuning(1, 0, 0, 0, False, 4)
    res["legacy_dyn_us"] = round(med_ts(lambda: fused_backward(dy, x, sc, mu, rs, out=out, workspace=ws, deterministic=False)), 2)
    res["legacy_det_us"] = round(med_ts(lambda: fused_backward(dy, x, sc, mu, rs, out=out, workspace=ws, deterministic=True)), 2)
    nat.set_tuning(1, 0, 0, 0, False, 0)
    res["steal_gbs"] = round(bb / res["steal_us"] / 1e3, 1)
    print(json.dumps(res), flush=True)
    del x, dy, mu, rs, out, ws
