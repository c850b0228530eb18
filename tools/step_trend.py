#!/usr/bin/env python3
"""Per-step fwd / bwd device times over a long fwd+bwd loop at cfg2 (bench.py's step), to see
how the forward's time evolves from the first steps after idle to steady state.

    python tools/step_trend.py [steps] [idle_s]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 400
idle = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
S, D = 32760, 5120
dev = torch.device("cuda", 0)
x = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
dy = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
sc = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
sh = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
st = torch.cuda.current_stream()
for _ in range(5):
    y, mu, rs = fused_forward(x, sc, sh)
    fused_backward(dy, x, sc, mu, rs)
torch.cuda.synchronize()
time.sleep(idle)
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
for k in range(steps):
    ev[k][0].record(st)
    y, mu, rs = fused_forward(x, sc, sh)
    ev[k][1].record(st)
    fused_backward(dy, x, sc, mu, rs)
    ev[k][2].record(st)
torch.cuda.synchronize()
f = [round(e[0].elapsed_time(e[1]) * 1e3, 1) for e in ev]
b = [round(e[1].elapsed_time(e[2]) * 1e3, 1) for e in ev]
print(json.dumps({"what": "fwd+bwd loop", "idle_s": idle, "fwd_us": f, "bwd_us": b}))
# forward-only loop, same buffers
torch.cuda.synchronize()
time.sleep(idle)
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
for k in range(steps):
    ev[k][0].record(st)
    y, mu, rs = fused_forward(x, sc, sh)
    ev[k][1].record(st)
torch.cuda.synchronize()
f = [round(e[0].elapsed_time(e[1]) * 1e3, 1) for e in ev]
print(json.dumps({"what": "fwd-only loop", "idle_s": idle, "fwd_us": f}))
