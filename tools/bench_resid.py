#!/usr/bin/env python3
"""Fused gated residual + AdaLN forward vs the unfused composition the reference's block runs
(x + gate * f in torch, then the AdaLN forward), one JSON line per shape.

Algorithmic bytes (fused): read x, f; write x_out, y  = 4 N D e  (+ 8 N stats + 3 B D e mods).
The unfused pair moves 2 N D e (torch mul: read f, write g*f) + 3 N D e (add) + 2 N D e (norm)
= 7 N D e with torch's eager mul+add, or 5 N D e with a single fused add; the fused kernel's
speed-up is measured, the bytes explain it.  Inputs (>= 2 x 300 MB) exceed the 126 MB L2.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln._ops import (fused_forward,  # noqa: E402
                                              fused_gate_residual_forward)


def timed(fn, iters=40):
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


def main():
    dev = torch.device("cuda", 0)
    shapes = [(1, 32760, 5120), (4, 8190, 5120), (8, 9450, 1536), (2, 32760, 1536)]
    if len(sys.argv) > 1:  # B,S,D ...
        shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
    for B, S, D in shapes:
        x = torch.randn(B, S, D, device=dev, dtype=torch.bfloat16)
        f = torch.randn_like(x)
        gate = 0.3 * torch.randn(B, D, device=dev, dtype=torch.bfloat16)
        sc = 0.1 * torch.randn(B, D, device=dev, dtype=torch.bfloat16)
        sh = 0.1 * torch.randn(B, D, device=dev, dtype=torch.bfloat16)
        nd = B * S * D * 2
        fused = timed(lambda: fused_gate_residual_forward(x, f, gate, sc, sh))
        eager = timed(lambda: fused_forward(x + f * gate[:, None, :], sc, sh))
        xo = torch.empty_like(x)
        addcmul = timed(lambda: fused_forward(torch.addcmul(x, f, gate[:, None, :], out=xo), sc, sh))
        print(json.dumps({
            "shape": [B, S, D], "dtype": "bf16",
            "fused_us": round(fused * 1e6, 1), "eager_mul_add_us": round(eager * 1e6, 1),
            "addcmul_us": round(addcmul * 1e6, 1),
            "fused_GBps": round((4 * nd + 8 * B * S) / fused / 1e9, 1),
            "speedup_vs_eager": round(eager / fused, 3), "speedup_vs_addcmul": round(addcmul / fused, 3),
        }))
        del x, f, xo
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
