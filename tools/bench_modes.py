#!/usr/bin/env python3
"""cfg2 fwd+bwd step time under four timing modes: eager with per-kernel events (round-1
bench.py), eager with only start/end events, one captured step replayed K times with per-kernel
external event nodes, the same without inner events.

    python tools/bench_modes.py [K] [W]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_17923_b200.adaln._ops import (  # noqa: E402
    backward_workspace_bytes, fused_backward, fused_forward)

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
import os  # noqa: E402
TAG = os.environ.get("AL_PDL_MASK", "default")
W = int(sys.argv[2]) if len(sys.argv) > 2 else 5
S, D = 32760, 5120
dev = torch.device("cuda", 0)
x = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
dy = torch.randn(1, S, D, device=dev).to(torch.bfloat16)
sc = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
sh = (0.1 * torch.randn(1, D, device=dev)).to(torch.bfloat16)
nbytes = 1677907520
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
EX = lambda: torch.cuda.Event(enable_timing=True, external=True)  # noqa: E731  (graph event nodes)


def step():
    y, mu, rs = fused_forward(x, sc, sh)
    return fused_backward(dy, x, sc, mu, rs)


def report(name, total_ms, fwd=None, bwd=None):
    d = {"mode": name, "pdl": TAG, "K": K, "ms_step": round(total_ms / K, 5),
         "gbs": round(nbytes / (total_ms / K * 1e-3) / 1e9, 1)}
    if fwd:
        d["fwd_us"] = round(1e3 * sum(fwd) / K, 2)
        d["bwd_us"] = round(1e3 * sum(bwd) / K, 2)
    print(json.dumps(d), flush=True)


st = torch.cuda.current_stream()
for rep in range(2):
    # (a) eager, per-kernel events
    for _ in range(W):
        step()
    torch.cuda.synchronize()
    ev = [[E() for _ in range(3)] for _ in range(K)]
    a, b = E(), E()
    a.record()
    for k in range(K):
        ev[k][0].record()
        y, mu, rs = fused_forward(x, sc, sh)
        ev[k][1].record()
        fused_backward(dy, x, sc, mu, rs)
        ev[k][2].record()
    b.record()
    torch.cuda.synchronize()
    report("eager+inner_events", a.elapsed_time(b), [e[0].elapsed_time(e[1]) for e in ev],
           [e[1].elapsed_time(e[2]) for e in ev])
    # (b) eager, outer events only
    for _ in range(W):
        step()
    torch.cuda.synchronize()
    a.record()
    for k in range(K):
        step()
    b.record()
    torch.cuda.synchronize()
    report("eager", a.elapsed_time(b))
    # (c)/(d) one captured step replayed
    for inner in (True, False):
        g = torch.cuda.CUDAGraph()
        evs = [EX() for _ in range(3)] if inner else None
        s2 = torch.cuda.Stream()
        s2.wait_stream(st)
        with torch.cuda.stream(s2):
            step()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s2):
                if inner:
                    evs[0].record()
                y, mu, rs = fused_forward(x, sc, sh)
                if inner:
                    evs[1].record()
                fused_backward(dy, x, sc, mu, rs)
                if inner:
                    evs[2].record()
        torch.cuda.synchronize()
        for _ in range(W):
            g.replay()
        torch.cuda.synchronize()
        a.record()
        for k in range(K):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        report("graph_step" + ("+inner_events" if inner else ""), a.elapsed_time(b))
    # (e) K steps in one graph over caller-owned buffers, per-kernel event nodes, uploaded first
    y = torch.empty_like(x)
    mu = torch.empty(1, S, device=dev)
    rs = torch.empty(1, S, device=dev)
    dx = torch.empty_like(x)
    dsc = torch.empty(1, D, device=dev)
    dsh = torch.empty(1, D, device=dev)
    ws = torch.empty(backward_workspace_bytes(x, sc), dtype=torch.uint8, device=dev)

    def step_into():
        fused_forward(x, sc, sh, out=y, out_mean=mu, out_rstd=rs)
        fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws)

    for _ in range(W):
        step_into()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    evk = [[EX() for _ in range(3)] for _ in range(K)]
    s2 = torch.cuda.Stream()
    s2.wait_stream(st)
    with torch.cuda.stream(s2):
        with torch.cuda.graph(g, stream=s2):
            for k in range(K):
                evk[k][0].record()
                fused_forward(x, sc, sh, out=y, out_mean=mu, out_rstd=rs)
                evk[k][1].record()
                fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws)
                evk[k][2].record()
    torch.cuda.synchronize()
    try:
        import cuda.bindings.runtime as rt
        err = rt.cudaGraphUpload(g.raw_cuda_graph_exec(), st.cuda_stream)
        upl = str(err[0] if isinstance(err, tuple) else err)
    except Exception as exc:  # noqa: BLE001
        upl = f"{type(exc).__name__}: {exc}"
    torch.cuda.synchronize()
    for _ in range(W):
        step_into()
    torch.cuda.synchronize()
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    report("graph_K_steps+inner_events (" + upl[:40] + ")", a.elapsed_time(b),
           [e[0].elapsed_time(e[1]) for e in evk], [e[1].elapsed_time(e[2]) for e in evk])
