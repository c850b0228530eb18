#!/usr/bin/env python3
"""Backward GB/s (graph-replayed chain of 20, L2-rotated inputs) per (vecs_per_thread, rows_per_stage)
tuning at short sequences, D=5120 bf16:  python tools/bwd_tuning_probe.py S [S ...]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

L2 = 126 << 20
dev = torch.device("cuda", 0)
for S in [int(a) for a in sys.argv[1:]] or [1560, 3600, 7800]:
    copies = max(1, -(-3 * L2 // (S * 5120 * 4)))
    sets = []
    for _ in range(copies):
        x = torch.randn(1, S, 5120, device=dev).to(torch.bfloat16)
        sc = (0.1 * torch.randn(1, 5120, device=dev)).to(torch.bfloat16)
        _, mu, rs = fused_forward(x, sc, sc)
        sets.append((torch.randn_like(x), x, sc, mu, rs))
    nb = 3 * S * 5120 * 2
    for V, R in ((0, 0), (1, 2), (1, 4), (2, 1), (2, 4), (4, 1)):
        nat.set_tuning(1, vecs_per_thread=V, rows_per_stage=R)
        try:
            for i in range(3):
                fused_backward(*sets[i % copies])
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                with torch.cuda.graph(g):
                    for i in range(20):
                        fused_backward(*sets[i % copies])
            torch.cuda.current_stream().wait_stream(st)
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) / 20 * 1e3
            plan = nat.describe_launch(1, 1, S, 5120, 5120, nat.AL_BF16)
            print(json.dumps({"S": S, "V": V, "R": R, "us": round(us, 2),
                              "gbs": round(nb / us / 1e3, 1), "plan": plan}), flush=True)
        finally:
            nat.set_tuning(1)
