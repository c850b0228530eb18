#!/usr/bin/env python3
"""Where the time goes at short sequences (cfg3 S = 1560 ... 14040, D = 5120 bf16): forward,
backward with the separate stage-2 kernel (variant 0) and with the fused cooperative stage 2
(variant 2), each replayed from a CUDA graph over L2-rotated inputs.  One JSON line per case."""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import adaln_bytes  # noqa: E402
from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

L2 = 126 << 20


def graph_ms(fn, copies, iters=20):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(g):
            for i in range(iters):
                fn(i)
    torch.cuda.current_stream().wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    dev = torch.device("cuda", 0)
    D = 5120
    for S in (1560, 3600, 7800, 14040):
        per = S * D * 2 * 2
        copies = max(1, -(-3 * L2 // per))
        sets = []
        for _ in range(copies):
            x = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
            sc = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
            dy = torch.randn_like(x)
            _, mu, rs = fused_forward(x, sc, sc)
            sets.append((x, sc, dy, mu, rs))
        nb = adaln_bytes(S, D, 1, 2)
        res = {"S": S, "copies": copies}
        res["fwd_us"] = 1e3 * graph_ms(lambda i: fused_forward(sets[i % copies][0], sets[i % copies][1],
                                                                sets[i % copies][1]), copies)
        for v in (0, 2):
            nat.set_tuning(1, variant=v)
            try:
                ms = graph_ms(lambda i: fused_backward(sets[i % copies][2], sets[i % copies][0],
                                                       sets[i % copies][1], sets[i % copies][3],
                                                       sets[i % copies][4]), copies)
            finally:
                nat.set_tuning(1)
            res[f"bwd_v{v}_us"] = 1e3 * ms
        res["fwd_gbs"] = nb["fwd"] / res["fwd_us"] / 1e3
        res["bwd_v0_gbs"] = nb["bwd"] / res["bwd_v0_us"] / 1e3
        res["bwd_v2_gbs"] = nb["bwd"] / res["bwd_v2_us"] / 1e3
        print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()}),
              flush=True)


if __name__ == "__main__":
    main()
