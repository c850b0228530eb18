#!/usr/bin/env python3
"""Backward-only chains (eager, back to back) vs fwd+bwd chains at several S, D=5120 bf16."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from bench import adaln_bytes  # noqa: E402
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402


def t(fn, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


dev = torch.device("cuda", 0)
for S in [int(a) for a in sys.argv[1:]] or [14040, 32760]:
    x = torch.randn(1, S, 5120, device=dev).to(torch.bfloat16)
    dy = torch.randn_like(x)
    sc = (0.1 * torch.randn(1, 5120, device=dev)).to(torch.bfloat16)
    _, mu, rs = fused_forward(x, sc, sc)
    nb = adaln_bytes(S, 5120)
    r = {"S": S}
    for det in (True, False):
        us = t(lambda: fused_backward(dy, x, sc, mu, rs, deterministic=det))
        r[f"bwd_chain_{'det' if det else 'dyn'}_gbs"] = round(nb["bwd"] / us / 1e3, 1)

    def step(det):
        _, m, s_ = fused_forward(x, sc, sc)
        fused_backward(dy, x, sc, m, s_, deterministic=det)
    for det in (True, False):
        us = t(lambda: step(det))
        r[f"fwdbwd_chain_{'det' if det else 'dyn'}_gbs"] = round(nb["total"] / us / 1e3, 1)
    print(json.dumps(r), flush=True)
