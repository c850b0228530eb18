#!/usr/bin/env python3
"""PCIe ceiling for the e2e leg: pinned host <-> device copy bandwidth of 335 MB (one cfg2 bf16
tensor) one direction at a time and both directions at once (two streams), CUDA events, best of
5.  The e2e step moves 671 MB each way (x and dy in; y and dx out), so 671 MB / (duplex GB/s)
bounds the step time the host API can reach."""
import json

import torch

n = 32760 * 5120
dev = torch.device("cuda", 0)
h_in = torch.empty(n, dtype=torch.bfloat16).pin_memory()
h_out = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d_in = torch.empty(n, dtype=torch.bfloat16, device=dev)
d_out = torch.randn(n, device=dev).to(torch.bfloat16)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
nb = n * 2


def best(fn, reps=5):
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out)


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t_h2d, t_d2h, t_both = best(h2d), best(d2h), best(both)
r = {"bytes": nb, "h2d_gbs": round(nb / t_h2d / 1e6, 1), "d2h_gbs": round(nb / t_d2h / 1e6, 1),
     "duplex_gbs_total": round(2 * nb / t_both / 1e6, 1),
     "cfg2_e2e_ceiling_gbs": round(1677.9e6 / (2 * t_both * 1e-3) / 1e9, 1)}
print(json.dumps(r))
