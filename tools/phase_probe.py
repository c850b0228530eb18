#!/usr/bin/env python3
"""Do the slow/fast phases of the cfg2 forward (tools/step_trend.py) also show up in plain torch
copy / add loops (i.e. a property of the box's HBM, not of the kernel)?  Runs several loops of
`steps` iterations back to back and prints per-20-step medians of each kernel's time.

    python tools/phase_probe.py [steps]
"""
import json
import statistics as stt
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 600
S, D = 32760, 5120
dev = torch.device("cuda", 0)
x = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
dy = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
o = torch.empty_like(x)
o2 = torch.empty_like(x)
sc = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
sh = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
st = torch.cuda.current_stream()
nd = S * D * 2


def loop(name, fns, nbytes):
    for _ in range(5):
        for f in fns:
            f()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(fns) + 1)] for _ in range(steps)]
    clk = torch.zeros(steps // 20 + 1, 2, dtype=torch.int64, device=dev)
    for k in range(steps):
        if k % 20 == 10:  # SM clock between two kernels, once per 20-step window
            nat.clock_probe(clk[k // 20].data_ptr(), 20000, st.cuda_stream)
        for j, f in enumerate(fns):
            ev[k][j].record(st)
            f()
        ev[k][-1].record(st)
    torch.cuda.synchronize()
    c = clk.cpu().tolist()
    out = {"loop": name, "sm_mhz_per20": [round(b / a * 1e3) if a else None for a, b in c[:steps // 20]]}
    for j in range(len(fns)):
        us = [e[j].elapsed_time(e[j + 1]) * 1e3 for e in ev]
        meds = [round(stt.median(us[i:i + 20]), 1) for i in range(0, steps, 20)]
        out[f"k{j}_gbs_med"] = round(nbytes[j] / (stt.median(us) * 1e-6) / 1e9, 1)
        out[f"k{j}_med20_us"] = meds
    print(json.dumps(out), flush=True)


_, mu, rs = fused_forward(x, sc, sh)
fb = 2 * nd + 8 * S
bb = 3 * nd + 8 * S
loop("copy+add", [lambda: o.copy_(x), lambda: torch.add(x, dy, out=o2)], [2 * nd, 3 * nd])
loop("fwd+bwd", [lambda: fused_forward(x, sc, sh), lambda: fused_backward(dy, x, sc, mu, rs)], [fb, bb])
loop("fwd(out=o)+bwd", [lambda: fused_forward(x, sc, sh, out=o), lambda: fused_backward(dy, x, sc, mu, rs)], [fb, bb])
loop("copy", [lambda: o.copy_(x)], [2 * nd])
loop("fwd", [lambda: fused_forward(x, sc, sh)], [fb])
loop("copy+add", [lambda: o.copy_(x), lambda: torch.add(x, dy, out=o2)], [2 * nd, 3 * nd])
loop("fwd+bwd", [lambda: fused_forward(x, sc, sh), lambda: fused_backward(dy, x, sc, mu, rs)], [fb, bb])
