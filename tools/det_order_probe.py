#!/usr/bin/env python3
"""Why does bench.py's deterministic-backward leg read slower than a fresh-process measurement?
cfg2, device timestamps: the deterministic backward issued eagerly (as bench.py's det leg) first
in the process, then after 20 graph-replayed + 20 eager default steps (bench.py's order), then
graph-replayed; and the default backward the same ways.  One JSON line."""

import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import (backward_workspace_bytes, fused_backward,  # noqa: E402
                                              fused_forward)

S, D, K = 32760, 5120, 20
dev = torch.device("cuda", 0)
x = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
dy = torch.randn_like(x)
sc = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
sh = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
y, dx = torch.empty_like(x), torch.empty_like(x)
mu, rs = torch.empty(1, S, device=dev), torch.empty(1, S, device=dev)
dsc, dsh = torch.empty(1, D, device=dev), torch.empty(1, D, device=dev)
ws = torch.empty(backward_workspace_bytes(x, sc), dtype=torch.uint8, device=dev)
ts = torch.empty(4 * K, 2, dtype=torch.int64, device=dev)


def step(det):
    fused_forward(x, sc, sh, out=y, out_mean=mu, out_rstd=rs)
    fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=det)


def eager(det):
    for _ in range(5):
        step(det)
    ts[:, 0] = -1
    ts[:, 1] = 0
    torch.cuda.synchronize()
    nat.set_timestamps(ts.data_ptr(), 4 * K)
    for _ in range(K):
        step(det)
    torch.cuda.synchronize()
    nat.set_timestamps(None)
    t = ts[:2 * K].cpu().tolist()
    return round(statistics.median([(e - b) / 1e3 for b, e in t[1::2]]), 2)


def graphed(det):
    for _ in range(5):
        step(det)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    ts[:, 0] = -1
    ts[:, 1] = 0
    torch.cuda.synchronize()
    nat.set_timestamps(ts.data_ptr(), 4 * K)
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for _ in range(K):
                step(det)
    nat.set_timestamps(None)
    for _ in range(5):
        step(det)
    ts[:, 0] = -1
    ts[:, 1] = 0
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    t = ts[:2 * K].cpu().tolist()
    return round(statistics.median([(e - b) / 1e3 for b, e in t[1::2]]), 2)


out = {"det_eager_first": eager(True), "dyn_graph": graphed(False), "dyn_eager": eager(False),
       "det_eager_after": eager(True), "det_graph": graphed(True), "dyn_eager_last": eager(False)}
print(json.dumps(out))
