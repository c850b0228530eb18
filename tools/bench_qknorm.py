#!/usr/bin/env python3
"""Fused Q/K RMSNorm (fwd, bwd) vs the torch path the block used before (split + nn.RMSNorm on
bf16 activations with fp32 weights -> the composite fp32 implementation), one JSON line per shape.
Algorithmic bytes: fwd reads q, k, v slices and writes q_n, k_n, v (6 N D e); bwd reads q, k, dq,
dk, dv and writes dq, dk, dv (8 N D e)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln import qk_rmsnorm  # noqa: E402


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e-3


def main():
    dev = torch.device("cuda", 0)
    d = 1536
    nq = torch.nn.RMSNorm(d, eps=1e-6).to(dev)
    nk = torch.nn.RMSNorm(d, eps=1e-6).to(dev)
    for lead in ((1, 32760), (20, 1560)):
        qkv = torch.randn(*lead, 3 * d, device=dev, dtype=torch.bfloat16, requires_grad=True)
        g = [torch.randn(*lead, d, device=dev, dtype=torch.bfloat16) for _ in range(3)]
        n = qkv.numel() // (3 * d)
        nde = n * d * 2

        def fused_fb():
            q, k, v = qk_rmsnorm(qkv, nq.weight, nk.weight)
            torch.autograd.backward([q, k, v], g)

        def torch_fb():
            q, k, v = qkv.split(d, dim=-1)
            q, k = nq(q).to(v.dtype), nk(k).to(v.dtype)
            torch.autograd.backward([q, k, v], g)

        def fused_f():
            with torch.no_grad():
                qk_rmsnorm(qkv, nq.weight, nk.weight)

        def torch_f():
            with torch.no_grad():
                q, k, v = qkv.split(d, dim=-1)
                nq(q).to(v.dtype), nk(k).to(v.dtype), v.contiguous()

        tf, tt = timed(fused_f), timed(torch_f)
        tfb, ttb = timed(fused_fb), timed(torch_fb)
        print(json.dumps({"rows": n, "D": d, "dtype": "bf16",
                          "fwd_fused_us": round(tf * 1e6, 1), "fwd_torch_us": round(tt * 1e6, 1),
                          "fwd_fused_GBps": round(6 * nde / tf / 1e9, 1),
                          "fwd_bwd_fused_us": round(tfb * 1e6, 1), "fwd_bwd_torch_us": round(ttb * 1e6, 1),
                          "fwd_bwd_fused_GBps": round(14 * nde / tfb / 1e9, 1),
                          "speedup_fwd": round(tt / tf, 2), "speedup_fwd_bwd": round(ttb / tfb, 2)}),
              flush=True)
        qkv.grad = None


if __name__ == "__main__":
    main()
