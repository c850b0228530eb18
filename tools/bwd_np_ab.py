#!/usr/bin/env python3
"""Producer-less backward (bwd_np.cuh: 12 warps x V=2 or 8 warps x V=3) vs K2 (adaln_bwd_tma, 11 warps): backward device
time (per-launch %globaltimer stamps, median of K eager launches after warm-up) at single-sample
lengths, dynamic and deterministic, plus a parity check of the selected kernel against a torch
fp64 restatement and run-to-run bit-identity of the deterministic mode.  AL_BWD_NP is read once
per process, so run it once per setting:

    for m in 0 12 8; do AL_BWD_NP=$m python tools/bwd_np_ab.py; done
"""
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import (backward_workspace_bytes, fused_backward,  # noqa: E402
                                              fused_forward)

D, K = 5120, 20
dev = torch.device("cuda", 0)
lens = [int(a) for a in sys.argv[1:]] or [14040, 20280, 32760, 46800, 75600]
tag = ",".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("AL_BWD")) or "default"
for S in lens:
    g = torch.Generator(device=dev).manual_seed(S)
    x = torch.randn(1, S, D, device=dev, generator=g).to(torch.bfloat16)
    dy = torch.randn(1, S, D, device=dev, generator=g).to(torch.bfloat16)
    sc = (0.1 * torch.randn(1, D, device=dev, generator=g)).to(torch.bfloat16)
    sh = (0.1 * torch.randn(1, D, device=dev, generator=g)).to(torch.bfloat16)
    y, mu, rs = fused_forward(x, sc, sh)
    dx = torch.empty_like(x)
    dsc = torch.empty(1, D, device=dev)
    dsh = torch.empty(1, D, device=dev)
    ws = torch.empty(backward_workspace_bytes(x, sc), dtype=torch.uint8, device=dev)
    out = {"S": S, "env": tag}
    nbytes = 3 * S * D * 2 + 8 * S + D * 2 + 8 * D
    for det in (False, True):
        for _ in range(5):
            fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=det)
        ts = torch.empty(K, 2, dtype=torch.int64, device=dev)
        ts[:, 0] = -1
        ts[:, 1] = 0
        torch.cuda.synchronize()
        nat.set_timestamps(ts.data_ptr(), K)
        for _ in range(K):
            fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=det)
        torch.cuda.synchronize()
        nat.set_timestamps(None)
        us = [(e - b) * 1e-3 for b, e in ts.cpu().tolist()]
        m = statistics.median(us)
        key = "det" if det else "dyn"
        out[key + "_us"] = round(m, 2)
        out[key + "_gbs"] = round(nbytes / (m * 1e-6) / 1e9, 1)
    # parity (deterministic result) against torch fp64
    fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=True)
    a = (dsc.clone(), dsh.clone(), dx.clone())
    fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=True)
    out["det_bitwise"] = bool(torch.equal(a[0], dsc) and torch.equal(a[1], dsh) and torch.equal(a[2], dx))
    xd, dyd = x.double()[0], dy.double()[0]
    xh = (xd - mu.double()[0, :, None]) * rs.double()[0, :, None]
    gg = dyd * (1 + sc.double())
    rdsc = (dyd * xh).sum(0)
    rdsh = dyd.sum(0)
    rdx = rs.double()[0, :, None] * (gg - gg.mean(1, keepdim=True) - xh * (gg * xh).mean(1, keepdim=True))
    rel = lambda u, r: float((u.double() - r).abs().max() / r.abs().max())  # noqa: E731
    out["rel_dscale"] = rel(dsc[0], rdsc)
    out["rel_dshift"] = rel(dsh[0], rdsh)
    out["rel_dx"] = rel(dx[0], rdx)
    fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=False)
    out["dyn_rel_dscale"] = rel(dsc[0], rdsc)
    out["dyn_rel_dx"] = rel(dx[0], rdx)
    print(json.dumps(out), flush=True)
    del x, dy, y, dx, ws
    torch.cuda.empty_cache()
