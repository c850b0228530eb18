#!/usr/bin/env python3
"""Timeline of the host-buffer e2e step (cfg2) with CUDA events around every chunk's upload,
kernels and download -- the same stream structure as adaln/_host.py (uploads + kernels on the
current stream, downloads on a side stream) -- to see where the step's time goes: per call the
first upload and the last download run alone (one PCIe direction idle).  Prints one JSON line
per call with the copy-engine busy times and the exposed (single-direction) time."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln import _host  # noqa: E402
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

dev = torch.device("cuda", 0)
S, D = 32760, 5120
xh = torch.randn(1, S, D).to(torch.bfloat16).pin_memory()
dyh = torch.randn(1, S, D).to(torch.bfloat16).pin_memory()
sc = (0.1 * torch.randn(1, D)).to(torch.bfloat16).pin_memory()
yh = torch.empty_like(xh).pin_memory()
dxh = torch.empty_like(xh).pin_memory()
muh = torch.empty(1, S).pin_memory()
rsh = torch.empty(1, S).pin_memory()
main = torch.cuda.current_stream()
side = torch.cuda.Stream()
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def call(kind, xdev):
    t0 = ev()
    t0.record(main)
    marks = []
    scd = sc.to(dev, non_blocking=True)
    for b0, b1, s0, s1 in _host._chunks(1, S, D * 2):
        a, b, c = ev(), ev(), ev()
        a.record(main)
        src = (xh if kind == "fwd" else dyh)[:, s0:s1]
        dd = torch.empty((1, s1 - s0, D), dtype=torch.bfloat16, device=dev)
        dd.copy_(src, non_blocking=True)
        b.record(main)
        if kind == "fwd":
            xdev[:, s0:s1].copy_(dd)
            out, mu, rs = fused_forward(dd, scd, scd)
        else:
            mud = torch.zeros(1, s1 - s0, device=dev)
            out, _, _ = fused_backward(dd, xdev[:, s0:s1], scd, mud + 0.0, mud + 1.0, deterministic=True)
        c.record(main)
        side.wait_stream(main)
        d, e = ev(), ev()
        with torch.cuda.stream(side):
            d.record(side)
            (yh if kind == "fwd" else dxh)[:, s0:s1].copy_(out, non_blocking=True)
            e.record(side)
        out.record_stream(side)
        marks.append((a, b, c, d, e))
    side.synchronize()
    torch.cuda.synchronize()
    rel = lambda x: t0.elapsed_time(x)  # noqa: E731
    h2d = [(rel(a), rel(b)) for a, b, c, d, e in marks]
    k = [(rel(b), rel(c)) for a, b, c, d, e in marks]
    d2h = [(rel(d), rel(e)) for a, b, c, d, e in marks]
    end = max(x[1] for x in d2h)
    return {"call": kind, "chunks": len(marks), "total_ms": round(end, 3),
            "h2d_busy_ms": round(sum(b - a for a, b in h2d), 3),
            "d2h_busy_ms": round(sum(b - a for a, b in d2h), 3),
            "kernel_ms": round(sum(b - a for a, b in k), 3),
            "first_h2d_ms": [round(v, 3) for v in h2d[0]], "last_d2h_ms": [round(v, 3) for v in d2h[-1]],
            "h2d_end_ms": round(h2d[-1][1], 3), "d2h_start_ms": round(d2h[0][0], 3)}


xdev = torch.empty(1, S, D, dtype=torch.bfloat16, device=dev)
for _ in range(3):
    call("fwd", xdev)
    call("bwd", xdev)
for _ in range(2):
    t = time.perf_counter()
    f = call("fwd", xdev)
    b = call("bwd", xdev)
    f["wall_step_ms"] = b["wall_step_ms"] = round(1e3 * (time.perf_counter() - t), 3)
    print(json.dumps(f))
    print(json.dumps(b))
