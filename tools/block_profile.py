#!/usr/bin/env python3
"""Kernel-time breakdown of one Wan-style DiT block fwd+bwd (the DP step's compute) with
torch.profiler (CUPTI), at a long-video and an image-like shape.  Prints the top kernels by
CUDA time and the share of our own (al::) kernels."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2605_17923_b200.dp_step import BlockConfig, WanStyleBlock  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    blk = WanStyleBlock(BlockConfig()).to(dev)
    for B, S in ((1, 32760), (20, 1560)):
        x = torch.randn(B, S, 1536, device=dev, dtype=torch.bfloat16)
        t = torch.randn(B, 1536, device=dev)
        tgt = torch.randn_like(x)

        def step():
            with torch.autocast("cuda", dtype=torch.bfloat16):
                o = blk(x, t)
                loss = F.mse_loss(o.float(), tgt.float())
            loss.backward()

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            for _ in range(3):
                step()
            torch.cuda.synchronize()
        kern, ops = [], []
        total = 0.0
        for ev in prof.key_averages():
            if ev.device_type == torch.autograd.DeviceType.CUDA:
                us = ev.device_time_total
                if us > 0:
                    total += us
                    kern.append((us, ev.count, ev.key))
            else:
                us = ev.self_device_time_total
                if us > 0:
                    ops.append((us, ev.count, ev.key))
        kern.sort(reverse=True)
        ops.sort(reverse=True)
        ours = sum(us for us, _, k in kern if "al::adaln" in k or "al::gate_res" in k)
        print(json.dumps({"B": B, "S": S, "ms_per_step": round(total / 3 / 1e3, 3),
                          "adaln_share": round(ours / total, 4),
                          "top_ops": [{"us_per_step": round(us / 3, 1), "calls": n // 3, "op": k[:60]}
                                      for us, n, k in ops[:25]],
                          "top_kernels": [{"us_per_step": round(us / 3, 1), "calls": n // 3,
                                           "kernel": k[:100]} for us, n, k in kern[:12]]},
                         indent=1), flush=True)


if __name__ == "__main__":
    main()
