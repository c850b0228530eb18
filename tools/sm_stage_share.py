#!/usr/bin/env python3
"""Stages per SM of the real backward (trace build: AB_NVCC_FLAGS=-DAL_CTA_TRACE
tools/ab_variant.sh trace <csrc-dir>; run with AL_LIB_VARIANT=trace).  In the dynamic (ticket)
walk a CTA's stage count measures its SM's sustained rate; compare with the traffic-only ticket
walk of tools/sm_topology_probe.cu to see whether the consumers cap the fast SMs."""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 32760
D = 5120
dev = torch.device("cuda", 0)
x = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
dy = torch.randn_like(x)
sc = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
sh = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
lib = ctypes.CDLL(str(nat.LIB_PATH))
lib.al_debug_cta_info.argtypes = [ctypes.c_void_p, ctypes.c_int]
y, mu, rs = fused_forward(x, sc, sh)
per_sm = np.zeros((0, 148))
for rep in range(24):
    fused_backward(dy, x, sc, mu, rs)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 4096)()
    assert lib.al_debug_cta_info(buf, 4096) == 0
    a = np.frombuffer(buf, dtype=np.uint64)[:148]
    row = np.zeros(148)
    for v in a:
        row[int(v >> 32) % 148] = int(v & 0xffffffff)
    if rep >= 2:
        per_sm = np.vstack([per_sm, row])
m = per_sm.mean(0)
print(json.dumps({"S": S, "stages_total": float(m.sum()), "per_sm_mean": [round(float(v), 1) for v in m],
                  "min": float(m.min()), "max": float(m.max())}))
