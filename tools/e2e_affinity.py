#!/usr/bin/env python3
"""Does host-thread / pinned-buffer NUMA placement move the e2e (host-buffer) number?

Measures pinned H2D/D2H bandwidth and the public-API fwd+bwd on host tensors (cfg2) twice:
with the process's default CPU affinity, and after restricting it to the GPU's NUMA-local cores
(NVML) and re-allocating the pinned buffers there (first touch).  Prints one JSON line each,
plus the topology facts used."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln import adaln_backward_naive, adaln_forward  # noqa: E402


def gpu_local_cpus(index: int = 0):
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(index)
    n = os.cpu_count() or 1
    words = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
    cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if m >> b & 1}
    return sorted(c for c in cpus if c < n)


def measure(tag):
    dev = torch.device("cuda", 0)
    S, D = 32760, 5120
    xh = torch.randn(1, S, D).to(torch.bfloat16).pin_memory()
    dyh = torch.randn(1, S, D).to(torch.bfloat16).pin_memory()
    sc = (0.1 * torch.randn(1, D)).to(torch.bfloat16).pin_memory()
    xd = xh.to(dev)
    oh = torch.empty_like(xh).pin_memory()
    nb = xh.numel() * 2

    def wall(fn, n=5):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) / n

    res = {"tag": tag, "affinity": len(os.sched_getaffinity(0))}
    res["h2d_GBs"] = round(nb / wall(lambda: xd.copy_(xh, non_blocking=True)) / 1e9, 2)
    res["d2h_GBs"] = round(nb / wall(lambda: oh.copy_(xd, non_blocking=True)) / 1e9, 2)

    def step():
        out = adaln_forward(xh, sc, sc, 1e-6, check_finite=False)
        adaln_backward_naive(dyh, xh, sc, out.mu, out.rstd, check_finite=False)

    for _ in range(3):
        step()
    total = 5 * nb + 8 * S  # fwd 2ND + bwd 3ND (bf16) + stats; algorithmic, as bench.py
    times = []
    for _ in range(6):
        torch.cuda.synchronize()
        t = time.perf_counter()
        step()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t)
    res["e2e_GBs_steps"] = [round(total / s / 1e9, 1) for s in times]
    print(json.dumps(res), flush=True)


def main():
    cpus = gpu_local_cpus(0)
    print(json.dumps({"os_cpus": os.cpu_count(), "gpu0_local_cpus": len(cpus),
                      "first": cpus[:4], "last": cpus[-4:]}), flush=True)
    measure("default")
    os.sched_setaffinity(0, cpus)
    measure("gpu-local")


if __name__ == "__main__":
    main()
