#!/usr/bin/env python3
"""PCIe reference points for the e2e (host-buffer) path: pinned H2D, D2H, both at once, and the
public API's forward / backward on pinned host tensors (cfg2)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln import adaln_backward_naive, adaln_forward  # noqa: E402

dev = torch.device("cuda", 0)
S, D = 32760, 5120
xh = torch.randn(1, S, D).to(torch.bfloat16).pin_memory()
dyh = torch.randn(1, S, D).to(torch.bfloat16).pin_memory()
sc = torch.zeros(1, D, dtype=torch.bfloat16).pin_memory()
xd = xh.to(dev)
oh = torch.empty_like(xh).pin_memory()
side = torch.cuda.Stream()
nb = xh.numel() * 2


def wall(fn, n=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n


res = {}
res["h2d_GBs"] = nb / wall(lambda: xd.copy_(xh, non_blocking=True)) / 1e9
res["d2h_GBs"] = nb / wall(lambda: oh.copy_(xd, non_blocking=True)) / 1e9


def both():
    xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(side):
        oh.copy_(yd, non_blocking=True)


yd = torch.empty_like(xd)
res["h2d_plus_d2h_concurrent_GBs"] = 2 * nb / wall(both) / 1e9
state = {}


def fwd():
    state["o"] = adaln_forward(xh, sc, sc, 1e-6, check_finite=False)


res["api_forward_ms"] = 1e3 * wall(fwd)
o = state["o"]
res["api_backward_ms"] = 1e3 * wall(lambda: adaln_backward_naive(dyh, xh, sc, o.mu, o.rstd,
                                                                  check_finite=False))
print(json.dumps({k: round(v, 2) for k, v in res.items()}))
