#!/usr/bin/env python3
"""Host-buffer (e2e) path at cfg2: PCIe reference rates and the public API's forward / backward
wall time per call for several pipeline chunk sizes (adaln._host.CHUNK_BYTES)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln import _host, adaln_backward_naive, adaln_forward  # noqa: E402

dev = torch.device("cuda", 0)
S, D = 32760, 5120
xh = torch.randn(1, S, D).to(torch.bfloat16).pin_memory()
dyh = torch.randn(1, S, D).to(torch.bfloat16).pin_memory()
sc = (0.1 * torch.randn(1, D)).to(torch.bfloat16).pin_memory()
xd = xh.to(dev)
yd = torch.empty_like(xd)
oh = torch.empty_like(xh).pin_memory()
side = torch.cuda.Stream()
nb = xh.numel() * 2


def wall(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n


def both():
    xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(side):
        oh.copy_(yd, non_blocking=True)
    torch.cuda.current_stream().wait_stream(side)


res = {"h2d_GBs": nb / wall(lambda: xd.copy_(xh, non_blocking=True)) / 1e9,
       "d2h_GBs": nb / wall(lambda: oh.copy_(xd, non_blocking=True)) / 1e9,
       "h2d_plus_d2h_concurrent_GBs": 2 * nb / wall(both) / 1e9}
print(json.dumps({k: round(v, 2) for k, v in res.items()}), flush=True)
alg = 1677907840
for mb in [int(a) for a in (sys.argv[1:] or ["8", "16", "32", "64"])]:
    _host.CHUNK_BYTES = mb << 20
    st = {}

    def fwd():
        st["o"] = adaln_forward(xh, sc, sc, 1e-6, check_finite=False)

    f = wall(fwd)
    o = st["o"]
    b = wall(lambda: adaln_backward_naive(dyh, xh, sc, o.mu, o.rstd, check_finite=False))
    print(json.dumps({"chunk_MB": mb, "api_forward_ms": round(1e3 * f, 2),
                      "api_backward_ms": round(1e3 * b, 2),
                      "e2e_GBs": round(alg / (f + b) / 1e9, 2)}), flush=True)
