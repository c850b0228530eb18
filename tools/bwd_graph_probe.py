#!/usr/bin/env python3
"""Backward-only chains replayed from a CUDA graph (20 launches) vs eager, S=14040 D=5120 bf16;
checks the replayed results against a deterministic eager call."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 14040
dev = torch.device("cuda", 0)
x = torch.randn(1, S, 5120, device=dev).to(torch.bfloat16)
dy = torch.randn_like(x)
sc = (0.1 * torch.randn(1, 5120, device=dev)).to(torch.bfloat16)
_, mu, rs = fused_forward(x, sc, sc)
ref = fused_backward(dy, x, sc, mu, rs, deterministic=True)
nbytes = 3 * S * 5120 * 2
out = {"S": S}
for det in (True, False):
    outs = []
    for _ in range(3):
        fused_backward(dy, x, sc, mu, rs, deterministic=det)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        with torch.cuda.graph(g):
            for _ in range(20):
                outs.append(fused_backward(dy, x, sc, mu, rs, deterministic=det))
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / 100 * 1e3
    ok = all(torch.equal(o[0], ref[0]) for o in outs)
    err = max(float((o[1] - ref[1]).abs().max() / ref[1].abs().max()) for o in outs)
    out["det" if det else "dyn"] = {"us": round(us, 2), "gbs": round(nbytes / us / 1e3, 1),
                                    "dx_equal": ok, "dscale_rel": err}
print(json.dumps(out))
