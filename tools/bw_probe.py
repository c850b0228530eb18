#!/usr/bin/env python3
"""Achievable HBM bandwidth for the AdaLN access patterns on this GPU (same process, same
sizes): torch copy (1 read : 1 write, like the forward) and torch add (2 reads : 1 write, like
the backward), next to the fused kernels.  Reference points for `roofline.frac`."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402


def t(fn, iters=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e-3


dev = torch.device("cuda", 0)
S, D = 32760, 5120
x = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
dy = torch.randn_like(x)
o = torch.empty_like(x)
sc = torch.zeros(1, D, device=dev, dtype=torch.bfloat16)
nd = S * D * 2
res = {}
res["copy_1r1w"] = 2 * nd / t(lambda: o.copy_(x)) / 1e9
res["add_2r1w"] = 3 * nd / t(lambda: torch.add(x, dy, out=o)) / 1e9
_, mu, rs = fused_forward(x, sc, sc)
res["adaln_fwd"] = (2 * nd + 8 * S) / t(lambda: fused_forward(x, sc, sc)) / 1e9
res["adaln_bwd"] = (3 * nd + 8 * S) / t(lambda: fused_backward(dy, x, sc, mu, rs)) / 1e9
print(json.dumps({k: round(v, 1) for k, v in res.items()}))
