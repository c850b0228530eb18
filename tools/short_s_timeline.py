#!/usr/bin/env python3
"""Device timeline of the fused fwd+bwd at short sequences (cfg3, D = 5120 bf16): one CUDA graph
of K steps over L2-rotated input sets, every launch stamping its own [first CTA start, last CTA
end] (al_debug_set_timestamps).  Per S: median forward / backward span, the gaps fwd->bwd and
bwd->next fwd, and the graph's step time.  With AL_LIB_VARIANT=cta_trace (built with
-DAL_CTA_TRACE) also the per-CTA start/end spread of the last forward and backward launch.
  python tools/short_s_timeline.py [S ...]"""

from __future__ import annotations

import ctypes
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import adaln_bytes  # noqa: E402
from paper_2605_17923_b200 import _native as nat  # noqa: E402
from paper_2605_17923_b200.adaln._ops import (backward_workspace_bytes, fused_backward,  # noqa: E402
                                              fused_forward)

L2 = 126 << 20
D = int(__import__("os").environ.get("AL_PROBE_D", "5120"))  # feature width (AL_PROBE_D)


def cta_spread(lib, kernel, grid):
    buf = (ctypes.c_ulonglong * (2 * 4096))()
    if lib.al_debug_cta_trace(kernel, buf, 2 * 4096) != 0:
        return None
    a = np.frombuffer(buf, dtype=np.uint64)[: 2 * grid].astype(np.int64).reshape(grid, 2)
    t0 = a[:, 0].min()
    st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
    return {"grid": grid, "start_us_q": [round(float(q), 2) for q in np.quantile(st, [0, .5, .9, 1])],
            "end_us_q": [round(float(q), 2) for q in np.quantile(en, [0, .1, .5, .9, 1])],
            "busy_frac": round(float(np.sum(en - st)) / (grid * float(en.max())), 4)}


def run(S, K=30, det=False, B=1):
    dev = torch.device("cuda", 0)
    per = 5 * B * S * D * 2
    ncopy = max(1, -(-2 * L2 // per))
    g = torch.Generator(device=dev).manual_seed(S)
    xs = [torch.randn(B, S, D, device=dev, generator=g).to(torch.bfloat16) for _ in range(ncopy)]
    dys = [torch.randn(B, S, D, device=dev, generator=g).to(torch.bfloat16) for _ in range(ncopy)]
    sc = (0.1 * torch.randn(B, D, device=dev, generator=g)).to(torch.bfloat16)
    sh = (0.1 * torch.randn(B, D, device=dev, generator=g)).to(torch.bfloat16)
    ys = [torch.empty_like(xs[0]) for _ in range(ncopy)]
    dxs = [torch.empty_like(xs[0]) for _ in range(ncopy)]
    mu = torch.empty(B, S, device=dev)
    rs = torch.empty(B, S, device=dev)
    dsc = torch.empty(B, D, device=dev)
    dsh = torch.empty(B, D, device=dev)
    ws = torch.empty(backward_workspace_bytes(xs[0], sc), dtype=torch.uint8, device=dev)

    def step(i):
        c = i % ncopy
        fused_forward(xs[c], sc, sh, out=ys[c], out_mean=mu, out_rstd=rs)
        fused_backward(dys[c], xs[c], sc, mu, rs, out=(dxs[c], dsc, dsh), workspace=ws,
                       deterministic=det)

    ts = torch.empty(2 * K, 2, dtype=torch.int64, device=dev)
    for i in range(5):
        step(i)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    ts[:, 0] = -1
    ts[:, 1] = 0
    torch.cuda.synchronize()
    nat.set_timestamps(ts.data_ptr(), 2 * K)
    try:
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                for i in range(K):
                    step(i)
    finally:
        nat.set_timestamps(None)
    for i in range(5):
        step(i)
    ts[:, 0] = -1
    ts[:, 1] = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
    t = ts.cpu().numpy().astype(np.int64)
    fw, bw = t[0::2], t[1::2]
    fspan = (fw[:, 1] - fw[:, 0]) / 1e3
    bspan = (bw[:, 1] - bw[:, 0]) / 1e3
    gap_fb = (bw[:, 0] - fw[:, 1]) / 1e3
    gap_bf = (fw[1:, 0] - bw[:-1, 1]) / 1e3
    ab = adaln_bytes(B * S, D, B)
    fb, bb = ab['fwd'], ab['bwd']
    step_us = e0.elapsed_time(e1) * 1e3 / K
    med = statistics.median
    out = {"S": S, "B": B, "det": det, "step_us": round(step_us, 2),
           "fwd_us": round(med(fspan), 2), "bwd_us": round(med(bspan), 2),
           "gap_fwd_to_bwd_us": round(med(gap_fb), 2), "gap_bwd_to_fwd_us": round(med(gap_bf), 2),
           "fwd_gbs": round(fb / med(fspan) / 1e3, 1), "bwd_gbs": round(bb / med(bspan) / 1e3, 1),
           "step_gbs": round((fb + bb) / step_us / 1e3, 1),
           "fwd_plan": nat.describe_launch(0, B, S, D, D, nat.AL_BF16),
           "bwd_plan": nat.describe_launch(1, B, S, D, D, nat.AL_BF16)}
    lib = ctypes.CDLL(str(nat.LIB_PATH))
    if hasattr(lib, "al_debug_cta_trace"):
        lib.al_debug_cta_trace.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
        out["cta_fwd"] = cta_spread(lib, 0, out["fwd_plan"]["grid"])
        out["cta_bwd"] = cta_spread(lib, 1, out["bwd_plan"]["grid"])
    del graph
    return out


def main():
    args = sys.argv[1:]
    if args and args[0] == "--one":  # --one B S det(0/1)
        print(json.dumps(run(int(args[2]), K=10, det=bool(int(args[3])), B=int(args[1]))), flush=True)
        return
    if args and args[0] == "--bucket1":  # --bucket1 S det(0/1): one bucket, this process
        from paper_2605_17923_b200.scheduler import DualConstraint, dual_constraint_batch
        S = int(args[1])
        B = dual_constraint_batch(S, DualConstraint(480_000.0, 3e9, 2.0))[0]
        print(json.dumps(run(S, K=10, det=bool(int(args[2])), B=B)), flush=True)
        return
    if args and args[0] == "--buckets":
        # cfg3 as the sampler issues it: B = the reference's dual-constraint batch for each S
        # (DualConstraint(M_mem = 480 000 tokens, M_comp = 3e9, p = 2), cluster_sim.py:332-336)
        from paper_2605_17923_b200.scheduler import DualConstraint, dual_constraint_batch
        c = DualConstraint(480_000.0, 3e9, 2.0)
        for S in [int(a) for a in args[1:]] or [1560, 3600, 7800, 14040, 20280, 32760, 46800,
                                                 61200, 75600]:
            B = dual_constraint_batch(S, c)[0]
            for det in (False, True):
                print(json.dumps(run(S, K=10, det=det, B=B)), flush=True)
        return
    for S in [int(a) for a in args] or [1560, 3600, 7800, 14040, 32760]:
        print(json.dumps(run(S)), flush=True)


if __name__ == "__main__":
    main()
