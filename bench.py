#!/usr/bin/env python3
"""Benchmark: fused AdaLN-Modulate fwd+bwd GB/s at the Wan-2.1-14B shape (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload adaln|dit] [--seq 32760] [--dim 5120]

One "step" = one fused forward (y, mean, rstd) + one fused backward (dx + dscale/dshift two-stage
reduction) over one [1, S, D] bf16 sample whose inputs are resident in HBM.  ``value`` is the
algorithmic bytes moved (fwd 2ND*2 + 2D*2 + 2N*4, bwd 3ND*2 + D*2 + 2N*4 + 2D*4)
divided by the device time, summed over ranks (weak scaling: each rank owns its own sample; the
op has no collective).  x and dy are 335 MB each (> 126 MB L2), so no L2 flush is needed.

``--impl reference`` times the reference algorithm on the host CPU (oracle/ -- the C
restatement of the numba kernels, bit-identical to them) with all host threads, on a bounded
row sample of the same workload, in the same metric.

``--workload dit`` runs the balanced DiT-block data-parallel step (see paper_2605_17923_b200/dp_step.py).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent
NOMINAL_HBM_GBS = 8000.0  # B200 datasheet HBM3e bandwidth (north_star's "~8 TB/s peak")


def peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    return HBM_FALLBACK_GBS, "fallback"


def adaln_bytes(n_rows: int, d: int, batch: int = 1, esize: int = 2) -> dict:
    """Algorithmic HBM bytes of one fused fwd and one fused bwd."""
    nd = n_rows * d
    fwd = 2 * nd * esize + 2 * batch * d * esize + 2 * n_rows * 4
    bwd = 3 * nd * esize + batch * d * esize + 2 * n_rows * 4 + 2 * batch * d * 4
    return {"fwd": fwd, "bwd": bwd, "total": fwd + bwd}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, enabled: bool = True):
        self.index = index
        self.enabled = enabled
        self.proc = None
        self.lines = []
        self.thread = None

    def __enter__(self):
        if not self.enabled:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- dist helpers
def dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        backend = "gloo" if args.impl == "reference" else "nccl"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    elif args.impl != "reference":
        torch.cuda.set_device(local)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- CPU baseline
def cpu_reference_gbs(seq_rows: int, d: int, threads: int, reps: int, seed: int = 0):
    """Time the reference algorithm (oracle = C restatement of the numba kernels) on the host:
    the public-API path _as_f64 (cast + isfinite) + forward + backward_naive (dx + reduction)."""
    import numpy as np

    import oracle

    rng = np.random.default_rng(seed)
    # bf16 bit patterns of N(0,1) draws (what the GPU arm reads)
    f = rng.standard_normal((seq_rows, d), dtype=np.float32)
    x16 = (f.view(np.uint32) >> 16).astype(np.uint16)
    f = rng.standard_normal((seq_rows, d), dtype=np.float32)
    dy16 = (f.view(np.uint32) >> 16).astype(np.uint16)
    sc16 = ((0.1 * rng.standard_normal(d, dtype=np.float32)).view(np.uint32) >> 16).astype(np.uint16)
    sh16 = ((0.1 * rng.standard_normal(d, dtype=np.float32)).view(np.uint32) >> 16).astype(np.uint16)
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        x, _ = oracle.as_f64(x16, threads)
        sc, _ = oracle.as_f64(sc16, threads)
        sh, _ = oracle.as_f64(sh16, threads)
        y, mu, rstd = oracle.forward(x, sc, sh, 1e-6, threads)
        dy, _ = oracle.as_f64(dy16, threads)
        dx, dsc, dsh = oracle.backward_naive(dy, x, sc, mu, rstd, threads)
        best = min(best, time.perf_counter() - t0)
        del y, dx
    nbytes = adaln_bytes(seq_rows, d)["total"]
    return nbytes / best / 1e9, best


# ----------------------------------------------------------------------------- arms
def run_reference(args, world, rank):
    """--impl reference: the reference algorithm on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle

    threads = os.cpu_count() or 1
    rows = args.ref_rows
    if args.warmup > 0:
        cpu_reference_gbs(min(rows, 1024), args.dim, threads, 1)
    times = []
    nbytes = adaln_bytes(rows, args.dim)["total"]
    for _ in range(args.steps):
        _, t = cpu_reference_gbs(rows, args.dim, threads, 1)
        times.append(t)
    total = sum(times)
    value = nbytes * args.steps / total / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 (bf16 inputs upcast)",
        "data": "synthetic",
        "config": {"workload": f"AdaLN fwd+bwd, Wan-2.1-14B row shape D={args.dim}, "
                               f"bounded sample of {rows} of {args.seq} rows per step",
                   "global_batch": 1, "seq_len": args.seq, "dim": args.dim},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{rows} rows x D={args.dim}: _as_f64 + forward + "
                                   "backward_naive (oracle/adaln_oracle.c, bit-identical "
                                   "to _kernels_numba.py), per step"},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "oracle_threads": oracle.max_threads(),
    }
    print(json.dumps(line), flush=True)


METRIC = "AdaLN-Modulate fwd+bwd GB/s (% HBM peak), Wan-14B shape; 8-GPU imbalance %"


def step_stats(ms: list, nbytes: int, peak: float) -> dict:
    """Per-launch spread over the timed steps (CUDA events on the launching stream)."""
    med = statistics.median(ms)
    return {"median_ms": round(med, 5), "min_ms": round(min(ms), 5), "max_ms": round(max(ms), 5),
            "median_frac": round(nbytes / (med * 1e-3) / 1e9 / peak, 4)}


def imbalance_summary(world: int) -> dict:
    from paper_2605_17923_b200 import sampler as smp
    from paper_2605_17923_b200.catalogs import reference_default_catalog
    from paper_2605_17923_b200.scheduler import emit_plan

    out = {}
    cat, w, tb, dc = reference_default_catalog()
    for n in sorted({8, max(world, 2)}):
        r = smp.compare_policies(cat, w, emit_plan(cat, tb), emit_plan(cat, dc), n, 500, 42)
        out[f"ranks_{n}"] = {
            "compute_cv_equal_token_pct": round(r["equal_token"]["mean_compute_cv"], 3),
            "compute_cv_dual_pct": round(r["dual"]["mean_compute_cv"], 3),
            "sim_cv_step_equal_token": round(r["equal_token"]["mean_cv_step"], 4),
            "sim_cv_step_dual": round(r["dual"]["mean_cv_step"], 4),
        }
    out["source"] = ("sampler draws (bit-exact with the reference's run_experiment, default "
                     "catalog, seed 42, 500 steps); measured per-rank step imbalance: "
                     "--workload dit")
    return out


def run_ours(args, world, rank, local):
    import torch

    from paper_2605_17923_b200 import _native as nat
    from paper_2605_17923_b200.adaln import adaln_backward_naive, adaln_forward
    from paper_2605_17923_b200.adaln._ops import (backward_workspace_bytes, fused_backward,
                                                  fused_forward)

    dev = torch.device("cuda", local)
    S, D = args.seq, args.dim
    g = torch.Generator(device="cpu").manual_seed(1234 + rank)
    # generate on device (fast), inputs resident in HBM
    gd = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn(1, S, D, device=dev, generator=gd, dtype=torch.float32).to(torch.bfloat16)
    dy = torch.randn(1, S, D, device=dev, generator=gd, dtype=torch.float32).to(torch.bfloat16)
    sc = (0.1 * torch.randn(1, D, generator=g)).to(torch.bfloat16).to(dev)
    sh = (0.1 * torch.randn(1, D, generator=g)).to(torch.bfloat16).to(dev)
    nb = adaln_bytes(S, D)
    stream = torch.cuda.current_stream(dev)

    # caller-owned outputs / workspace, reused by every step (as a training loop's buffers)
    y = torch.empty_like(x)
    mu = torch.empty(1, S, device=dev)
    rs = torch.empty(1, S, device=dev)
    dx = torch.empty_like(x)
    dsc = torch.empty(1, D, device=dev)
    dsh = torch.empty(1, D, device=dev)
    ws = torch.empty(backward_workspace_bytes(x, sc), dtype=torch.uint8, device=dev)

    def step(det=False):
        fused_forward(x, sc, sh, out=y, out_mean=mu, out_rstd=rs)
        fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=det)

    K = args.steps
    # per-launch device timestamps (al_debug_set_timestamps): [start, end] of every fwd (K1) and
    # bwd (K2 start .. K3 end) launch, written by the kernels themselves -- an event record
    # between the two launches would break their PDL overlap and add ~5 us to each
    ts = torch.empty(4 * K, 2, dtype=torch.int64, device=dev)

    def ts_arm():
        ts[:, 0] = -1  # UINT64_MAX for the atomicMin of the start stamp
        ts[:, 1] = 0

    def ts_read(n):
        return [(e - b) * 1e-6 for b, e in ts[:n].cpu().tolist()]  # ms

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    # the timed steps: one CUDA graph of K steps (each the fwd + bwd launches of the public device
    # API, captured in order, so each launch keeps its own timestamp pair), uploaded before timing
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(stream)
    ts_arm()
    torch.cuda.synchronize(dev)
    nat.set_timestamps(ts.data_ptr(), 4 * K)
    try:
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                for _ in range(K):
                    step()
    finally:
        nat.set_timestamps(None)
    torch.cuda.synchronize(dev)
    try:
        import cuda.bindings.runtime as cudart

        cudart.cudaGraphUpload(graph.raw_cuda_graph_exec(), stream.cuda_stream)
    except Exception:  # noqa: BLE001 - the upload only moves the first replay's setup earlier
        pass
    torch.cuda.synchronize(dev)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local, enabled=not args.no_clocks) as clk:
        # the sampler's first nvidia-smi lines arrive before the GPU work starts; the warm-up
        # steps then run immediately before the timed region, so the first timed kernel does
        # not pay the ramp out of an idle power state (a 0.3 s idle gap before a 6 ms timed
        # region cost the driver's 20-step run +13 us on the average forward in round 1)
        time.sleep(0.3)
        for _ in range(args.warmup):
            step()
        ts_arm()
        barrier(world)
        torch.cuda.synchronize(dev)
        start.record(stream)
        graph.replay()
        end.record(stream)
        torch.cuda.synchronize(dev)
        barrier(world)
    elapsed_ms = start.elapsed_time(end)
    lt = ts_read(2 * K)
    fwd_ms, bwd_ms = lt[0::2], lt[1::2]
    del graph

    # the same K steps issued eagerly (one Python call per op, as a training loop issues them)
    for _ in range(args.warmup):
        step()
    ts_arm()
    torch.cuda.synchronize(dev)
    nat.set_timestamps(ts.data_ptr(), 4 * K)
    start.record(stream)
    for _ in range(K):
        step()
    end.record(stream)
    torch.cuda.synchronize(dev)
    nat.set_timestamps(None)
    eager_ms = start.elapsed_time(end)
    lt = ts_read(2 * K)
    eager_fwd, eager_bwd = lt[0::2], lt[1::2]

    # the reference-facing API's backward (adaln_backward_naive/_dtile force the static,
    # bit-reproducible partition): timed the same way (device timestamps), after the headline
    for _ in range(args.warmup):
        step(det=True)
    ts_arm()
    torch.cuda.synchronize(dev)
    nat.set_timestamps(ts.data_ptr(), 4 * K)
    for _ in range(K):
        step(det=True)
    torch.cuda.synchronize(dev)
    nat.set_timestamps(None)
    det_ms = ts_read(2 * K)[1::2]

    elapsed_ms = max_over_ranks(elapsed_ms, world)
    eager_ms = max_over_ranks(eager_ms, world)
    ms_step = elapsed_ms / K
    value = world * nb["total"] / (ms_step * 1e-3) / 1e9
    peak, peak_kind = peak_hbm()
    fwd_avg, bwd_avg = sum(fwd_ms) / K, sum(bwd_ms) / K
    bwd_gbs = nb["bwd"] / (bwd_avg * 1e-3) / 1e9
    fwd_gbs = nb["fwd"] / (fwd_avg * 1e-3) / 1e9

    # ---- e2e: the public API with pinned HOST buffers (H2D + D2H inside the timed region)
    xh = x.cpu().pin_memory()
    dyh = dy.cpu().pin_memory()
    sch, shh = sc.cpu().pin_memory(), sh.cpu().pin_memory()
    e2e_steps = max(1, min(K, args.e2e_steps))

    def e2e_step():
        out = adaln_forward(xh, sch, shh, 1e-6, check_finite=False)
        gr = adaln_backward_naive(dyh, xh, sch, out.mu, out.rstd, check_finite=False)
        return out, gr

    # warm-up: the pinned host result buffers come from the host API's pinned pool; two
    # generations are alive at once (previous step's results + this step's), so fill it; then
    # one full collection, so a generational GC pass over the warm-up's garbage does not land
    # inside the timed steps (tools/e2e_steps_diag.py: 95-170 ms steps 2-6 with GC, none without)
    import gc

    for _ in range(max(3, args.warmup)):
        out, gr = e2e_step()
    torch.cuda.synchronize(dev)
    gc.collect()
    barrier(world)
    t0 = time.perf_counter()
    step_s = []
    for _ in range(e2e_steps):
        ts = time.perf_counter()
        out, gr = e2e_step()  # returns after the D2H of its results completed
        step_s.append(time.perf_counter() - ts)
    torch.cuda.synchronize(dev)
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps, world)
    barrier(world)
    es = 2
    # forward: x, scale, shift in; y, mean, rstd out.  backward: dy (+ x unless the forward's
    # device copy of x is still valid -- the host API keeps it, _host.py), scale, mean, rstd in;
    # dx, dscale, dshift out
    from paper_2605_17923_b200.adaln._host import _resident

    x_again = 0 if _resident.enabled else x.numel() * es
    h2d = (x.numel() * es + 2 * D * es) + (x.numel() * es + x_again + D * es + 2 * S * 4)
    d2h = (x.numel() * es + 2 * S * 4) + (x.numel() * es + 2 * D * 4)
    e2e_gbs = world * nb["total"] / e2e_s / 1e9
    # the PCIe ceiling of that leg on this box: one cfg2 tensor host->device and another
    # device->host at the same time (two streams, pinned memory, best of 3); the host API moves
    # h2d + d2h bytes per step, so (h2d + d2h) / duplex rate bounds its step time
    pcie = None
    try:
        hb = torch.empty_like(xh, pin_memory=True)
        db = torch.empty_like(x)
        s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        best = float("inf")
        for _ in range(3):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            with torch.cuda.stream(s1):
                db.copy_(xh, non_blocking=True)
            with torch.cuda.stream(s2):
                hb.copy_(y, non_blocking=True)
            torch.cuda.synchronize(dev)
            best = min(best, time.perf_counter() - t0)
        duplex = 2 * xh.numel() * es / best / 1e9
        pcie = {"duplex_gbs": round(duplex, 1),
                "e2e_ceiling": round(world * nb["total"] / ((h2d + d2h) / (duplex * 1e9)) / 1e9, 1)
                if duplex > 0 else None}
        del hb, db
    except Exception as exc:  # noqa: BLE001 - informative only
        pcie = {"error": f"{type(exc).__name__}: {exc}"[:200]}

    # measured 'N-GPU imbalance %' of the metric: the DP step on this process group under
    # each bucket plan (equal token, the reference's dual constraint, the reference fitter's
    # power-law dual on B200 trials, the two-term time-balanced plan), N > 1 only
    dp = None
    if world > 1 and not args.no_dp:
        del x, dy, xh, dyh, out, gr, y, dx, ws
        torch.cuda.empty_cache()
        try:
            from paper_2605_17923_b200 import dp_step

            arms = tuple(a for a in args.dp_arms.split(",") if a)
            r = dp_step.run_arms(world, rank, local, steps=args.dp_steps, warmup=2, arms=arms,
                                 detail=False)
            dp = {"workload": r["config"]["workload"], "steps_per_policy": args.dp_steps,
                  "plans": r["config"]["plans"], "arms": r["config"]["arms"],
                  "imbalance": r["imbalance"],
                  "bottleneck": {a: r["policies"][a]["bottleneck"] for a in arms},
                  "measured_ms_by_bucket": {a: r["policies"][a]["measured_ms_by_bucket"]
                                            for a in arms},
                  "calibration": (None if not r["calibration"] else
                                  {k: r["calibration"][k] for k in ("power_fit", "quadratic_fit",
                                                                    "predicted_ms")})}
        except Exception as exc:  # noqa: BLE001 - the kernel line must still be printed
            dp = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if rank != 0:
        return
    # CPU baseline: the reference algorithm, single thread (as the numba reference runs)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        rows = args.cpu_rows
        gbs, t = cpu_reference_gbs(rows, D, 1, 2)
        cpu = {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "port",
               "sample": f"{rows} of {S} rows x D={D} (bf16 values upcast), _as_f64 + forward + "
                         f"backward_naive, best of 2 = {t:.2f} s (oracle/adaln_oracle.c, "
                         "bit-identical to the single-threaded numba reference)"}
    traffic = None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("bwd_dram_bytes_per_launch")
        except (ValueError, OSError):
            traffic = None
    fplan = nat.describe_launch(0, 1, S, D, D, nat.AL_BF16)
    bplan = nat.describe_launch(1, 1, S, D, D, nat.AL_BF16)
    line = {
        "metric": METRIC,
        "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"fused AdaLN-Modulate fwd+bwd, Wan-2.1-14B shape B=1 S={S} D={D} "
                               "bf16 per rank (BASELINE configs[1])",
                   "global_batch": world, "seq_len": S, "dim": D,
                   "parallelism": f"dp{world} (independent samples per rank; no collective in the op)",
                   "l2": "inputs larger than L2 (x, dy 335 MB each vs 126 MB L2); no flush",
                   "scheduling": "forward: dynamic row tail (bit-identical to a static split); "
                                 "backward: ticketed stage walk (dscale/dshift in a "
                                 "timing-dependent fp32 order, torch deterministic mode off); "
                                 "kernels.bwd_deterministic = the reference API's fixed "
                                 "interleaved walk",
                   "timing": "K steps (fused_forward + fused_backward of the public device API "
                             "into caller-owned buffers) captured in order into one CUDA graph, "
                             "replayed once between CUDA events; per-kernel times from the "
                             "kernels' own device timestamps (al_debug_set_timestamps) of the "
                             "same launches; value_eager = the same K steps issued eagerly"},
        "value_eager": round(world * nb["total"] / (eager_ms / K * 1e-3) / 1e9, 2),
        "ms_per_step_eager": round(eager_ms / K, 5),
        "pct_hbm_peak": round(100 * value / world / peak, 2),
        # north_star's "≥75 % of B200 HBM peak" against the nominal 8 TB/s as well
        "pct_nominal_peak": round(100 * value / world / NOMINAL_HBM_GBS, 2),
        "roofline": {"bound": "hbm", "kernel": "adaln_bwd (stage-1 adaln_bwd_tma + stage-2 reduce)",
                     "achieved": round(bwd_gbs, 1), "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(bwd_gbs / peak, 4), "traffic": traffic,
                     "bytes_per_launch": nb["bwd"], "avg_ms": round(bwd_avg, 5)},
        "kernels": {"fwd": {"gbs": round(fwd_gbs, 1), "frac": round(fwd_gbs / peak, 4),
                            "avg_ms": round(fwd_avg, 5), **step_stats(fwd_ms, nb["fwd"], peak),
                            "bytes": nb["fwd"], "plan": fplan},
                    "bwd": {"gbs": round(bwd_gbs, 1), "frac": round(bwd_gbs / peak, 4),
                            "avg_ms": round(bwd_avg, 5), **step_stats(bwd_ms, nb["bwd"], peak),
                            "bytes": nb["bwd"], "plan": bplan},
                    "bwd_deterministic": {
                        "gbs": round(nb["bwd"] / (sum(det_ms) / K * 1e-3) / 1e9, 1),
                        "frac": round(nb["bwd"] / (sum(det_ms) / K * 1e-3) / 1e9 / peak, 4),
                        "avg_ms": round(sum(det_ms) / K, 5), **step_stats(det_ms, nb["bwd"], peak),
                        "bytes": nb["bwd"],
                        "what": "fused_backward(deterministic=True): the partition the "
                                "reference-facing API (adaln_backward_naive/_dtile) runs; "
                                "dscale/dshift bit-identical run to run",
                        "plan": bplan},
                    "eager_fwd": {"avg_ms": round(sum(eager_fwd) / K, 5),
                                  **step_stats(eager_fwd, nb["fwd"], peak)},
                    "eager_bwd": {"avg_ms": round(sum(eager_bwd) / K, 5),
                                  **step_stats(eager_bwd, nb["bwd"], peak)},
                    "timer": "per-launch device timestamps (%globaltimer: first CTA start .. "
                             "last CTA end; the backward = stage 1 start .. stage 2 end)"},
        "e2e": {"value": round(e2e_gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "step_ms_min_max": [round(1e3 * min(step_s), 2), round(1e3 * max(step_s), 2)],
                "step_ms_median": round(1e3 * statistics.median(step_s), 2),
                "pcie": pcie,
                "path": "adaln_forward + adaln_backward_naive on pinned torch CPU bf16 tensors "
                        "(the backward reuses the forward's device copy of x)"
                        if _resident.enabled else
                        "adaln_forward + adaln_backward_naive on pinned torch CPU bf16 tensors"},
        "cpu_baseline": cpu,
        "gpu_launches": 3 * K,  # fwd K1 + bwd K2 + K3 per step (the deterministic leg is outside)
        "clocks": clk.summary(),
        "imbalance": imbalance_summary(world),
    }
    if dp is not None:
        line["dp_step"] = dp
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["adaln", "dit"], default="adaln")
    ap.add_argument("--seq", type=int, default=32760)
    ap.add_argument("--dim", type=int, default=5120)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-rows", type=int, default=8192)
    ap.add_argument("--ref-rows", type=int, default=8192)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-dp", action="store_true", help="skip the N>1 DP-step imbalance A/B")
    ap.add_argument("--dp-steps", type=int, default=16)
    ap.add_argument("--dp-arms", default="equal_token,dual_reference,dual_power_fit,dual_quadratic")
    args, rest = ap.parse_known_args()
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and args.impl == "ours":
        # NCCL communicator init lines (nRanks, NVLS / channels) for the driver's rank count;
        # NCCL reads these once, so they are set before anything imports torch
        # (set, not setdefault: images that export NCCL_DEBUG=WARN would silence them)
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
        # to stderr: NCCL logs to stdout by default, after the JSON line (which must stay the
        # last line of rank 0's stdout)
        os.environ["NCCL_DEBUG_FILE"] = "/dev/stderr"
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world, rank, local = dist_setup(args)
    try:
        if args.workload == "dit" and args.impl == "reference":
            if rank == 0:
                print(json.dumps({"impl": "reference", "unavailable":
                                  "the reference has no DiT step: its DP step is a simulated "
                                  "barrier (cluster_sim.py:134-158)"}), flush=True)
        elif args.workload == "dit":
            from paper_2605_17923_b200 import dp_step

            dp_step.bench_main(args, rest, world, rank, local)
        elif args.impl == "reference":
            run_reference(args, world, rank)
        else:
            run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
