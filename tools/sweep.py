#!/usr/bin/env python3
"""Launch-configuration sweep for the AdaLN kernels (CUDA-event timing, inputs > L2).

    python tools/sweep.py [--seq 32760] [--dim 5120] [--dtype bf16] [--iters 20]

Prints one JSON line per configuration with the kernel's achieved GB/s (algorithmic bytes /
average duration) and the fraction of MEASURED_PEAKS.json hbm_gbs.
"""

from __future__ import annotations

import argparse
import itertools
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import adaln_bytes, peak_hbm  # noqa: E402
from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward  # noqa: E402

DT = {"bf16": (torch.bfloat16, nat.AL_BF16, 2), "fp32": (torch.float32, nat.AL_F32, 4),
      "f16": (torch.float16, nat.AL_F16, 2)}


def time_fn(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=32760)
    ap.add_argument("--dim", type=int, default=5120)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--which", default="fwd,bwd")
    ap.add_argument("--variants", default="0,1,2,3,4,5,6", help="forward rows variants to time")
    ap.add_argument("--no-ring", action="store_true", help="skip the V/R/smem ring sweep")
    ap.add_argument("--ring7-cfgs", default="",
                    help="extra ring-forward configs 'V:R:smemKB,...' (variant 7)")
    ap.add_argument("--fwd-ring7", action="store_true",
                    help="sweep V/R/smem of the backward-style ring forward (variant 7)")
    args = ap.parse_args()
    dt, code, es = DT[args.dtype]
    B, S, D = args.batch, args.seq, args.dim
    dev = torch.device("cuda", 0)
    x = torch.randn(B, S, D, device=dev).to(dt)
    dy = torch.randn(B, S, D, device=dev).to(dt)
    sc = (0.1 * torch.randn(B, D, device=dev)).to(dt)
    sh = (0.1 * torch.randn(B, D, device=dev)).to(dt)
    nb = adaln_bytes(B * S, D, B, es)
    peak, _ = peak_hbm()
    _, mu, rs = fused_forward(x, sc, sh)

    def report(kind, cfg, ms, nbytes, plan):
        gbs = nbytes / (ms * 1e-3) / 1e9
        print(json.dumps({"kernel": kind, "cfg": cfg, "ms": round(ms, 5), "gbs": round(gbs, 1),
                          "frac": round(gbs / peak, 4), "plan": plan}), flush=True)

    if "fwd" in args.which:
        cfgs = [dict(variant=int(v)) for v in args.variants.split(",")]
        if not args.no_ring:
            cfgs += [dict(V=V, R=R, smem=sm) for V, R, sm in itertools.product(
                (1, 2, 4), (1, 2, 4), (100 * 1024, 200 * 1024))]
        for spec in filter(None, args.ring7_cfgs.split(",")):
            V, R, kb = (int(v) for v in spec.split(":"))
            cfgs.append(dict(V=V, R=R, smem=kb * 1024, variant=7))
        if args.fwd_ring7:
            cfgs += [dict(V=V, R=R, smem=sm, variant=7) for V, R, sm in itertools.product(
                (0, 1, 2, 4), (0, 1, 2, 4), (0, 100 * 1024, 200 * 1024))]
        for c in cfgs:
            try:
                nat.set_tuning(0, c.get("V", 0), c.get("R", 0), c.get("smem", 0), False,
                               c.get("variant", 0))
                plan = nat.describe_launch(0, B, S, D, D, code)
                ms = time_fn(lambda: fused_forward(x, sc, sh), args.iters)
                report("fwd", c, ms, nb["fwd"], plan)
            except Exception as exc:  # noqa: BLE001
                print(json.dumps({"kernel": "fwd", "cfg": c, "error": str(exc)[:200]}))
        nat.set_tuning(0)
    if "bwd" in args.which:
        cfgs = [dict(V=0, R=0, smem=0, variant=v) for v in (0, 2)]  # separate vs fused stage 2
        cfgs += [dict(V=V, R=R, smem=sm) for V, R, sm in itertools.product(
            (1, 2, 4), (1, 2, 4), (0, 100 * 1024, 150 * 1024, 200 * 1024))]
        for c in cfgs:
            try:
                nat.set_tuning(1, c["V"], c["R"], c["smem"], False, c.get("variant", 0))
                plan = nat.describe_launch(1, B, S, D, D, code)
                ms = time_fn(lambda: fused_backward(dy, x, sc, mu, rs), args.iters)
                report("bwd", c, ms, nb["bwd"], plan)
            except Exception as exc:  # noqa: BLE001
                print(json.dumps({"kernel": "bwd", "cfg": c, "error": str(exc)[:200]}))
        nat.set_tuning(1)


if __name__ == "__main__":
    main()
