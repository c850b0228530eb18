#!/usr/bin/env python3
"""Per-step wall time of the public host-buffer API (cfg2 fwd+bwd) with the pinned host
allocator's statistics after each step -- to see whether slow steps coincide with new
cudaHostAlloc calls."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln import adaln_backward_naive, adaln_forward  # noqa: E402


def stats():
    try:
        s = torch.cuda.host_memory_stats()
        return {k: s[k] for k in ("num_host_alloc", "num_host_free", "allocated_bytes.current",
                                  "reserved_bytes.current") if k in s} or {"keys": list(s)[:8]}
    except Exception as exc:  # noqa: BLE001
        return {"err": str(exc)[:80]}


S, D = 32760, 5120
xh = torch.randn(1, S, D).to(torch.bfloat16).pin_memory()
dyh = torch.randn(1, S, D).to(torch.bfloat16).pin_memory()
sc = (0.1 * torch.randn(1, D)).to(torch.bfloat16).pin_memory()
total = 5 * xh.numel() * 2 + 8 * S
out = gr = None
import gc  # noqa: E402

if "--no-gc" in sys.argv:
    gc.disable()
COLLECT_AT = 3 if "--collect" in sys.argv else -1
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 12):  # noqa: E501
    torch.cuda.synchronize()
    if i == COLLECT_AT:
        gc.collect()
    t = time.perf_counter()
    c = time.process_time()
    out = adaln_forward(xh, sc, sc, 1e-6, check_finite=False)
    t1 = time.perf_counter()
    gr = adaln_backward_naive(dyh, xh, sc, out.mu, out.rstd, check_finite=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(json.dumps({"step": i, "ms": round(dt * 1e3, 1), "fwd_ms": round((t1 - t) * 1e3, 1),
                      "cpu_ms": round((time.process_time() - c) * 1e3, 1),
                      "GBs": round(total / dt / 1e9, 1), **stats()}), flush=True)
