#!/usr/bin/env python3
"""Round-1 backward (tuning variant 4) at cfg2 with the ring depth forced to 3/4/5 stages via the
smem budget: how much the in-flight depth matters.  Device-timestamp medians."""
import json
import statistics as stt
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

dev = torch.device("cuda", 0)
S, D = 32760, 5120
x = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
dy = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
sc = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
_, mu, rs = fused_forward(x, sc, sc)
ts = torch.empty(30, 2, dtype=torch.int64, device=dev)
for ns in (3, 4, 5):
    for det in (False, True):
        nat.set_tuning(1, 0, 0, ns * 40960 + 2048, False, 4)
        for _ in range(3):
            fused_backward(dy, x, sc, mu, rs, deterministic=det)
        ts[:, 0] = -1
        ts[:, 1] = 0
        torch.cuda.synchronize()
        nat.set_timestamps(ts.data_ptr(), 30)
        for _ in range(30):
            fused_backward(dy, x, sc, mu, rs, deterministic=det)
        torch.cuda.synchronize()
        nat.set_timestamps(None)
        us = stt.median([(e - b) / 1e3 for b, e in ts.cpu().tolist()])
        print(json.dumps({"ns": ns, "det": det, "us": round(us, 2),
                          "plan": nat.describe_launch(1, 1, S, D, D, nat.AL_BF16)}), flush=True)
nat.set_tuning(1, 0, 0, 0, False, 0)
