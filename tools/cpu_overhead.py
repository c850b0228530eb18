#!/usr/bin/env python3
"""Host-side cost of one fused fwd+bwd call pair (Python + ctypes + allocator), no GPU sync."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

dev = torch.device("cuda", 0)
x = torch.randn(1, 64, 5120, device=dev).to(torch.bfloat16)
dy = torch.randn_like(x)
sc = torch.zeros(1, 5120, device=dev, dtype=torch.bfloat16)
for _ in range(10):
    y, mu, rs = fused_forward(x, sc, sc)
    fused_backward(dy, x, sc, mu, rs)
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for _ in range(n):
    y, mu, rs = fused_forward(x, sc, sc)
t1 = time.perf_counter()
for _ in range(n):
    fused_backward(dy, x, sc, mu, rs)
t2 = time.perf_counter()
torch.cuda.synchronize()
print(f"host us per fused_forward {1e6 * (t1 - t0) / n:.1f}, per fused_backward {1e6 * (t2 - t1) / n:.1f}")
