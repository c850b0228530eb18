#!/usr/bin/env python3
"""Per-CTA start/end spread of the forward (rows16) and backward (TMA ring) kernels at cfg2,
from a trace build (AB_NVCC_FLAGS=-DAL_CTA_TRACE tools/ab_variant.sh <name> <src>; run with
AL_LIB_VARIANT=<name>).  Prints, per kernel, the CTA start spread, the end-time quantiles
relative to the first start, and the share of the kernel span during which CTAs were idle."""
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
lib.al_debug_cta_trace.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
for _ in range(5):
    y, mu, rs = fused_forward(x, sc, sh)
    fused_backward(dy, x, sc, mu, rs)
torch.cuda.synchronize()
out = {"S": S, "lib": nat.LIB_PATH.name}
for k, name, grid in ((0, "fwd", nat.describe_launch(0, 1, S, D, D, nat.AL_BF16)["grid"]),
                      (1, "bwd", nat.describe_launch(1, 1, S, D, D, nat.AL_BF16)["grid"])):
    buf = (ctypes.c_ulonglong * (2 * 4096))()
    assert lib.al_debug_cta_trace(k, buf, 2 * 4096) == 0
    a = np.frombuffer(buf, dtype=np.uint64)[: 2 * grid].astype(np.int64).reshape(grid, 2)
    t0 = a[:, 0].min()
    st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
    span = en.max()
    busy = float(np.sum(en - st)) / (grid * span)
    out[name] = {"grid": int(grid), "span_us": round(float(span), 2),
                 "start_us_max": round(float(st.max()), 2),
                 "end_us_q": [round(float(q), 2) for q in np.quantile(en, [0, .1, .5, .9, 1])],
                 "busy_frac": round(busy, 4),
                 "slowest_ctas": [int(i) for i in np.argsort(-en)[:8]],
                 "fastest_ctas": [int(i) for i in np.argsort(en)[:8]]}
print(json.dumps(out))
