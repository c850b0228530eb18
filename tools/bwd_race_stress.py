#!/usr/bin/env python3
"""Stress the backward ring for a slot-reuse race: repeat the same launch N times and count
launches whose dx / dscale differ bitwise from the first (deterministic schedules must never
differ).  Shapes: a single-sample launch and a group-walk multi-sample launch; the release point
is AL_BWD_EARLY (read once per process).  One JSON line per shape."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln._ops import backward_workspace_bytes, fused_backward, fused_forward  # noqa: E402

dev = torch.device("cuda", 0)
n_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 200
shapes = [(1, 32760, 5120), (2, 20000, 2048), (2, 18000, 5120), (5, 17000, 1024)]
if os.environ.get("STRESS_ALL"):
    # + the short-launch pipeline kernel, auto work stealing (multi-sample short), wide rows
    shapes += [(1, 8000, 5120), (1, 3600, 1024), (3, 7001, 5120), (24, 1560, 5120),
               (4, 3000, 1536), (1, 12000, 8192)]
for b, s, d in shapes:
    g = torch.Generator(device="cpu").manual_seed(s)
    x = torch.randn(b, s, d, generator=g).to(torch.bfloat16).to(dev)
    dy = torch.randn(b, s, d, generator=g).to(torch.bfloat16).to(dev)
    sc = (0.1 * torch.randn(b, d, generator=g)).to(torch.bfloat16).to(dev)
    _, mu, rs = fused_forward(x, sc, sc)
    ref = [t.clone() for t in fused_backward(dy, x, sc, mu, rs, deterministic=True)]
    dx = torch.empty_like(x)
    dsc = torch.empty(b, d, device=dev)
    dsh = torch.empty(b, d, device=dev)
    ws = torch.empty(backward_workspace_bytes(x, sc), dtype=torch.uint8, device=dev)
    y0 = fused_forward(x, sc, sc)[0].clone()
    bad_y = 0
    for _ in range(max(1, n_iter // 5)):
        bad_y += int(not torch.equal(fused_forward(x, sc, sc)[0], y0))
    bad_dx = bad_dsc = 0
    worst = 0.0
    for i in range(n_iter):
        fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=True)
        if i % 10 == 9 or i == n_iter - 1:
            torch.cuda.synchronize()
        if not torch.equal(dx, ref[0]):
            bad_dx += 1
            worst = max(worst, float((dx.float() - ref[0].float()).abs().max()))
        if not torch.equal(dsc, ref[1]):
            bad_dsc += 1
    print(json.dumps({"shape": [b, s, d], "AL_BWD_EARLY": os.environ.get("AL_BWD_EARLY", "default"),
                      "iters": n_iter, "y_mismatches": bad_y, "dx_mismatches": bad_dx, "dscale_mismatches": bad_dsc,
                      "worst_dx_abs_diff": worst}), flush=True)
