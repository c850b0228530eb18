#!/usr/bin/env python3
"""Median device time of the fused forward and backward (dynamic and deterministic) over a few
BASELINE shapes; run once per library build (AL_LIB_VARIANT=<name> selects
_lib/variants/<name>.so) and compare the lines.

    AL_LIB_VARIANT=base python tools/ab_time.py [iters] [tag]
"""
import json
import os
import statistics as stt
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
tag = sys.argv[2] if len(sys.argv) > 2 else os.environ.get("AL_LIB_VARIANT", "tree")
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
D = 5120
clk = torch.zeros(1, 2, dtype=torch.int64, device=dev)


def med(fn, per_graph=10):
    """Device time per call: `per_graph` calls captured in one CUDA graph (so short kernels are
    not timed against the Python launch overhead), graph replays timed with events; median."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    s2.wait_stream(st)
    with torch.cuda.stream(s2):
        with torch.cuda.graph(gr, stream=s2):
            for _ in range(per_graph):
                fn()
    torch.cuda.synchronize()
    for _ in range(2):
        gr.replay()
    reps = max(3, iters // per_graph)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(reps)]
    for i in range(reps):
        ev[i][0].record(st)
        gr.replay()
        ev[i][1].record(st)
    torch.cuda.synchronize()
    return stt.median([a.elapsed_time(b) * 1e3 / per_graph for a, b in ev])


for B, S in [(1, 32760), (1, 1560), (1, 3600), (1, 7800), (4, 1560), (1, 75600)]:
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(B, S, D, device=dev, generator=g).to(torch.bfloat16)
    dy = torch.randn(B, S, D, device=dev, generator=g).to(torch.bfloat16)
    sc = (0.1 * torch.randn(B, D, device=dev, generator=g)).to(torch.bfloat16)
    _, mu, rs = fused_forward(x, sc, sc)
    fb = 2 * B * S * D * 2 + 2 * B * D * 2 + 8 * B * S
    bb = 3 * B * S * D * 2 + B * D * 2 + 8 * B * S + 8 * B * D
    f = med(lambda: fused_forward(x, sc, sc))
    bd = med(lambda: fused_backward(dy, x, sc, mu, rs, deterministic=False))
    bs = med(lambda: fused_backward(dy, x, sc, mu, rs, deterministic=True))
    extra = {}
    if os.environ.get("AB_LEGACY"):  # the round-1 scheme (tuning variant 4) in the same process
        nat.set_tuning(1, 0, 0, 0, False, 4)
        extra["legacy_dyn_us"] = round(med(lambda: fused_backward(dy, x, sc, mu, rs, deterministic=False)), 2)
        extra["legacy_det_us"] = round(med(lambda: fused_backward(dy, x, sc, mu, rs, deterministic=True)), 2)
        nat.set_tuning(1, 0, 0, 0, False, 0)
    nat.clock_probe(clk.data_ptr(), 20000, st.cuda_stream)
    c = clk.cpu().tolist()[0]
    print(json.dumps({"tag": tag, "B": B, "S": S, "fwd_us": round(f, 2), "bwd_dyn_us": round(bd, 2),
                      "bwd_det_us": round(bs, 2), "fwd_gbs": round(fb / f / 1e3, 1),
                      "bwd_dyn_gbs": round(bb / bd / 1e3, 1), "bwd_det_gbs": round(bb / bs / 1e3, 1),
                      "sm_mhz": round(c[1] / c[0] * 1e3), **extra}), flush=True)
    del x, dy, mu, rs
