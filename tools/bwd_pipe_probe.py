#!/usr/bin/env python3
"""A/B of the backward stage-1 kernels: adaln_bwd_tma (variant 0) vs the skewed-pipeline
adaln_bwd_pipe (variant 3, R = 1 / 2), static (deterministic) and dynamic tail, at cfg2 and the
short cfg3 lengths; median device time of `iters` back-to-back launches + agreement with the
default kernel's outputs.

    python tools/bwd_pipe_probe.py [iters]
"""
import json
import statistics as stt
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
D = 5120
cases = [(1, 32760), (1, 1560), (1, 3600), (1, 7800), (4, 1560), (1, 75600)]
variants = [("tma", 0, 0), ("pipe_R2", 3, 2), ("pipe_R1", 3, 1)]
clk = torch.zeros(1, 2, dtype=torch.int64, device=dev)
for B, S in cases:
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(B, S, D, device=dev, generator=g).to(torch.bfloat16)
    dy = torch.randn(B, S, D, device=dev, generator=g).to(torch.bfloat16)
    sc = (0.1 * torch.randn(B, D, device=dev, generator=g)).to(torch.bfloat16)
    sh = (0.1 * torch.randn(B, D, device=dev, generator=g)).to(torch.bfloat16)
    _, mu, rs = fused_forward(x, sc, sh)
    nb = 3 * B * S * D * 2 + B * D * 2 + 8 * B * S + 8 * B * D
    ref = None
    for name, var, R in variants:
        for det in (True, False):
            nat.set_tuning(1, 0, R, 0, False, var)
            out = fused_backward(dy, x, sc, mu, rs, deterministic=det)
            torch.cuda.synchronize()
            if ref is None:
                ref = [t.float() for t in out]
            err = [float((a.float() - b).abs().max() / b.abs().max().clamp_min(1e-30))
                   for a, b in zip(out, ref)]
            for _ in range(5):
                fused_backward(dy, x, sc, mu, rs, deterministic=det)
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(iters)]
            for i in range(iters):
                ev[i][0].record(st)
                fused_backward(dy, x, sc, mu, rs, deterministic=det)
                ev[i][1].record(st)
            nat.clock_probe(clk.data_ptr(), 20000, st.cuda_stream)
            torch.cuda.synchronize()
            us = stt.median([a.elapsed_time(b) * 1e3 for a, b in ev])
            c = clk.cpu().tolist()[0]
            print(json.dumps({"B": B, "S": S, "kernel": name, "deterministic": det,
                              "us": round(us, 2), "gbs": round(nb / us / 1e3, 1),
                              "sm_mhz": round(c[1] / c[0] * 1e3), "plan": nat.describe_launch(1, B, S, D, D, nat.AL_BF16),
                              "relerr_vs_tma_det": [f"{e:.1e}" for e in err]}), flush=True)
    nat.set_tuning(1, 0, 0, 0, False, 0)
    del x, dy, mu, rs
