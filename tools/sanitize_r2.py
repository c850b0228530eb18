#!/usr/bin/env python3
"""Small-shape driver for compute-sanitizer (one tool per run): every round-2 kernel path once --
rows16 forward with and without its dynamic tail, rows/rows2/ring/generic forwards, the lock-step
backward (dynamic tail, static, interleaved), the skewed-pipeline backward (static and dynamic),
the work-stealing backward (when AL_BWD_STEAL=1), both stage-2 kernels, the gated-residual
forward/backward (vector and generic), the Q/K RMSNorm pair."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import (fused_backward, fused_forward,  # noqa: E402
                                              fused_gate_residual_backward,
                                              fused_gate_residual_forward,
                                              fused_qk_rmsnorm_backward, fused_qk_rmsnorm_forward)

dev = torch.device("cuda", 0)
cases = [(2, 37, 1024, torch.bfloat16), (1, 129, 1536, torch.float32), (3, 9, 12288, torch.bfloat16),
         (2, 17, 5120, torch.bfloat16), (2, 5, 3, torch.float32), (1, 33, 2048, torch.float64),
         (1, 12000, 256, torch.bfloat16),   # dynamic tails (>= 64 rows per CTA in the tail)
         (1, 20000, 512, torch.float16)]    # > the short-launch limit: lock-step kernel
for b, s, d, dt in cases:
    x = torch.randn(b, s, d, device=dev).to(dt)
    dy = torch.randn_like(x)
    sc = (0.1 * torch.randn(b, d, device=dev)).to(dt)
    sh = (0.1 * torch.randn(b, d, device=dev)).to(dt)
    for fwd_variant in (0, 2, 7):
        nat.set_tuning(0, variant=fwd_variant)
        y, mu, rs = fused_forward(x, sc, sh, check_finite=True)
    nat.set_tuning(0)
    for det in (False, True):
        for bwd_variant, R in ((0, 0), (3, 2), (4, 0)):
            nat.set_tuning(1, rows_per_stage=R, variant=bwd_variant)
            fused_backward(dy, x, sc, mu, rs, check_finite=True, deterministic=det)
        # broadcast modulation: a single group (interleaved static partition when deterministic)
        nat.set_tuning(1)
        fused_backward(dy.view(-1, d), x.view(-1, d), sc[0], mu.view(-1), rs.view(-1),
                       deterministic=det)
    f = torch.randn_like(x)
    g = (0.1 * torch.randn(b, d, device=dev)).to(dt)
    xo, y2, m2, r2 = fused_gate_residual_forward(x, f, g, sc, sh)
    fused_gate_residual_backward(dy, dy, f, g)
    fused_gate_residual_backward(dy.view(-1)[: b * s * d].view(b, s, d), None, f, g)
    if d * x.element_size() <= 4096 and (d * x.element_size()) % 16 == 0:
        qkv = torch.randn(b, s, 3 * d, device=dev).to(dt)
        w = torch.ones(d, device=dev).to(dt)
        qn, kn, v, rq = fused_qk_rmsnorm_forward(qkv, w, w)
        fused_qk_rmsnorm_backward(qkv, w, w, rq, torch.randn_like(qn), torch.randn_like(kn), v)
# misaligned views: the generic kernels
buf = torch.randn(1 + 4 * 300, device=dev)
xm = buf[1:].view(4, 300)
fused_forward(xm, torch.zeros(300, device=dev), torch.zeros(300, device=dev))
gbuf = torch.randn(1 + 2 * 10 * 1000, device=dev).to(torch.bfloat16)
gm = gbuf[1:].view(2, 10, 1000)
fused_gate_residual_backward(gm, None, gm, torch.ones(2, 1000, device=dev).to(torch.bfloat16))
torch.cuda.synchronize()
print("sanitize driver ok")
