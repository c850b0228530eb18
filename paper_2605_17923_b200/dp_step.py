"""Data-parallel DiT-block training step fed by the bucket sampler (north-star subsystem 3).

The reference has no GPU step: it models the data-parallel barrier as T_sync = max_i T_i
(cluster_sim.py:134-158) over synthetic times.  This module runs the real thing on B200s:

* every rank builds the same ``BucketSampler`` (same seed) and takes shard ``rank`` of each
  step's draw -- bucket assignment needs no communication and is bit-identical to the
  reference's ``sample_assignments`` (cluster_sim.py:113-131);
* rank i runs forward + backward of a Wan-2.1-style DiT block on its synthetic batch
  [B_i, S_i, D] (fused AdaLN from ``adaln.FusedAdaLNModulate`` for both modulated norms;
  attention/GEMMs through torch, i.e. cuBLAS / flash SDPA);
* the only collective is ONE NCCL all-reduce of the flat fp32 gradient buffer at the step
  boundary (NVLink / NVSwitch), then a fused AdamW step;
* the per-rank compute time T_i (CUDA events, before the all-reduce) is all-gathered (a few
  bytes) to report the reference's imbalance metrics on measured times: cv_step = (max-min)/max
  (cluster_sim.py:161-166) and wait_sync = max T - T_i, next to compute_cv over B_i * S_i^2
  (cluster_sim.py:169-174).

Gradient averaging with heterogeneous per-rank batches is token-weighted: each rank's loss is
the sum of its per-token losses divided by the step's GLOBAL token count (known on every rank
from the shared draw), so the all-reduce SUM is exactly the global per-token mean gradient.

The block (Wan-2.1-1.3B widths: D=1536, 12 heads, FFN 8960) is public architecture, not part
of the reference; weights are random-initialised and the data synthetic.
"""

from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

from .errors import AdaptiveLoadError
from .sampler import BucketSampler, RankShard, compute_cv, cv_step
from .scheduler import emit_plan

__all__ = ["WanStyleBlock", "DPStepRunner", "StepStats", "bench_main"]


@dataclass(frozen=True)
class BlockConfig:
    dim: int = 1536
    heads: int = 12
    ffn: int = 8960
    eps: float = 1e-6


class WanStyleBlock(nn.Module):
    """AdaLN-modulated self-attention + FFN block with six per-sample modulation vectors.

    ``norm_fn(x, scale, shift, eps)`` is the fused LayerNorm-Modulate; the default is the
    sm_100a kernel pair (``adaln_modulate``).  Tests may inject a CPU stand-in to exercise the
    data-parallel host logic on gloo.  With the default norm the attention residual and the
    second norm run as ONE fused kernel (``gate_residual_adaln``: x + gate1 * proj(a) -> AdaLN),
    and Q/K RMSNorm reads q and k straight out of the qkv projection (``qk_rmsnorm``).
    """

    def __init__(self, cfg: BlockConfig = BlockConfig(), norm_fn=None):
        super().__init__()
        self.cfg = cfg
        d = cfg.dim
        self.modulation = nn.Parameter(torch.randn(1, 6, d) / math.sqrt(d))
        self.time_proj = nn.Linear(d, 6 * d)
        self.qkv = nn.Linear(d, 3 * d)
        # Wan-2.1 norm_q / norm_k: RMSNorm over the full width of q and k
        self.q_norm = nn.RMSNorm(d, eps=cfg.eps)
        self.k_norm = nn.RMSNorm(d, eps=cfg.eps)
        self.proj = nn.Linear(d, d)
        self.ffn_in = nn.Linear(d, cfg.ffn)
        self.ffn_out = nn.Linear(cfg.ffn, d)
        self.resid_norm_fn = None
        self.qk_norm_fn = None
        if norm_fn is None:
            from .adaln import adaln_modulate, gate_residual_adaln, qk_rmsnorm

            norm_fn = adaln_modulate
            self.resid_norm_fn = gate_residual_adaln
            self.qk_norm_fn = qk_rmsnorm
        self.norm_fn = norm_fn

    def forward(self, x: torch.Tensor, t_emb: torch.Tensor) -> torch.Tensor:
        b, s, d = x.shape
        h = self.cfg.heads
        e = (self.time_proj(F.silu(t_emb)).view(b, 6, d) + self.modulation).to(x.dtype)
        shift1, scale1, gate1, shift2, scale2, gate2 = e.unbind(1)
        y = self.norm_fn(x, scale1.contiguous(), shift1.contiguous(), self.cfg.eps)
        qkv = self.qkv(y)
        # the fused Q/K norm holds a whole row in one warp's registers: rows of <= 4 KB (bf16
        # D <= 2048, the Wan-1.3B width); wider blocks (Wan-14B D = 5120) take nn.RMSNorm
        if self.qk_norm_fn is not None and d * qkv.element_size() <= 4096:
            q, k, v = self.qk_norm_fn(qkv, self.q_norm.weight, self.k_norm.weight, self.cfg.eps)
        else:
            q, k, v = qkv.split(d, dim=-1)
            q, k = self.q_norm(q).to(v.dtype), self.k_norm(k).to(v.dtype)
        q, k, v = (t.view(b, s, h, d // h).transpose(1, 2) for t in (q, k, v))
        a = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(b, s, d)
        if self.resid_norm_fn is not None:
            x, y = self.resid_norm_fn(x, self.proj(a), gate1.contiguous(), scale2.contiguous(),
                                      shift2.contiguous(), self.cfg.eps)
        else:
            x = x + self.proj(a) * gate1[:, None, :]
            y = self.norm_fn(x, scale2.contiguous(), shift2.contiguous(), self.cfg.eps)
        x = x + self.ffn_out(F.gelu(self.ffn_in(y), approximate="tanh")) * gate2[:, None, :]
        return x


@dataclass
class StepStats:
    step: int
    shards: list
    t_compute_ms: list      # measured T_i per rank (fwd+bwd, before the all-reduce)
    t_step_ms: float        # max over ranks of the full step (incl. all-reduce + optimizer)
    tokens: int             # sum of B_i * S_i
    loads: list             # B_i * S_i^2
    cv_step: float          # (max - min) / max over measured T_i
    compute_cv: float       # 100 * std / mean over B_i * S_i^2
    wait_sync_ms: list      # max T - T_i

    def to_json(self) -> dict:
        return {"step": self.step, "seq": [sh.seq_len for sh in self.shards],
                "batch": [sh.batch_size for sh in self.shards],
                "t_compute_ms": [round(t, 4) for t in self.t_compute_ms],
                "t_step_ms": round(self.t_step_ms, 4), "tokens": self.tokens,
                "cv_step": self.cv_step, "compute_cv": self.compute_cv}


class DPStepRunner:
    """One DP rank: shard -> synthetic batch -> fwd/bwd -> one flat all-reduce -> AdamW."""

    def __init__(self, block: nn.Module, device: torch.device, world: int, rank: int,
                 dtype=torch.bfloat16, lr: float = 1e-4, seed: int = 0, group=None):
        self.block = block.to(device)
        self.device = device
        self.world, self.rank = world, rank
        self.dtype = dtype
        self.group = group
        self.params = [p for p in self.block.parameters() if p.requires_grad]
        numel = sum(p.numel() for p in self.params)
        # one contiguous fp32 gradient buffer: the all-reduce is a single NCCL call
        self.flat_grad = torch.zeros(numel, dtype=torch.float32, device=device)
        off = 0
        for p in self.params:
            p.grad = self.flat_grad[off:off + p.numel()].view_as(p)
            off += p.numel()
        fused = device.type == "cuda"
        self.opt = torch.optim.AdamW(self.params, lr=lr, fused=fused)
        self.gen = torch.Generator(device=device).manual_seed(seed * 1000 + rank)
        self.dim = block.cfg.dim

    def make_batch(self, shard: RankShard):
        b, s, d = shard.batch_size, shard.seq_len, self.dim
        x = torch.randn(b, s, d, device=self.device, generator=self.gen, dtype=self.dtype)
        t = torch.randn(b, d, device=self.device, generator=self.gen, dtype=self.dtype)
        target = torch.randn(b, s, d, device=self.device, generator=self.gen, dtype=self.dtype)
        return x, t, target

    def _allreduce(self, t: torch.Tensor):
        if self.world > 1:
            import torch.distributed as dist

            dist.all_reduce(t, group=self.group)

    def _all_gather_scalar(self, v: float) -> list:
        if self.world == 1:
            return [v]
        import torch.distributed as dist

        dev = self.device if dist.get_backend(self.group) == "nccl" else torch.device("cpu")
        outs = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(self.world)]
        dist.all_gather(outs, torch.tensor([v], dtype=torch.float64, device=dev), group=self.group)
        return [float(a.item()) for a in outs]

    def step(self, step_idx: int, shards: list, batch=None) -> StepStats:
        mine = shards[self.rank]
        global_tokens = sum(sh.tokens for sh in shards)
        x, t, target = batch if batch is not None else self.make_batch(mine)
        cuda = self.device.type == "cuda"
        if cuda:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
        else:
            t0 = time.perf_counter()
        self.flat_grad.zero_()
        with torch.autocast(self.device.type, dtype=torch.bfloat16, enabled=cuda):
            out = self.block(x, t)
            # token-weighted: per-token MSE summed locally, normalised by the GLOBAL token count
            loss = F.mse_loss(out.float(), target.float(), reduction="sum") / (
                global_tokens * self.dim)
        loss.backward()
        if cuda:
            ev[1].record()
        else:
            t1 = time.perf_counter()
        self._allreduce(self.flat_grad)
        self.opt.step()
        if cuda:
            ev[2].record()
            torch.cuda.synchronize(self.device)
            t_comp = ev[0].elapsed_time(ev[1])
            t_step = ev[0].elapsed_time(ev[2])
        else:
            t_comp = 1e3 * (t1 - t0)
            t_step = 1e3 * (time.perf_counter() - t0)
        times = self._all_gather_scalar(t_comp)
        t_step_max = max(self._all_gather_scalar(t_step))
        loads = [sh.load for sh in shards]
        return StepStats(step_idx, shards, times, t_step_max, global_tokens, loads,
                         cv_step(times), compute_cv(loads) if len(loads) > 1 else 0.0,
                         [max(times) - v for v in times])


def measure_trials(runner: DPStepRunner, requests, reps: int = 3) -> list:
    """Time one rank's fwd+bwd for each (B, S) request (CUDA events, median of `reps` after a
    warm-up); returns costfit.Trial records in seconds -- the B200 counterpart of the
    reference's synthetic sweep (costfit.generate_sweep + cluster_sim ground truth)."""
    from .costfit import Trial
    from .shapes import Bucket, MediaShape

    out = []
    for b, s in requests:
        shard = RankShard(runner.rank, -1, Bucket(MediaShape(1, 16, 16), s, 1), b)
        batch = runner.make_batch(shard)
        times = []
        for _ in range(reps + 1):
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            runner.flat_grad.zero_()
            with torch.autocast("cuda", dtype=torch.bfloat16):
                o = runner.block(batch[0], batch[1])
                loss = F.mse_loss(o.float(), batch[2].float())
            loss.backward()
            ev1.record()
            torch.cuda.synchronize(runner.device)
            times.append(ev0.elapsed_time(ev1) / 1e3)
        out.append(Trial(b, s, float(np.median(times[1:]))))
        del batch, o, loss
    return out


def calibrate_plan(runner: DPStepRunner, catalog, m_mem: float, cost_model: str = "quadratic"):
    """Sweep -> fit -> plan every bucket to the longest bucket's B=1 time.

    cost_model "power": the reference's T = a + b B S^p (grid-searched p) and its dual
    constraint; "quadratic": T = a + c1 B S + c2 B S^2 (costfit.time_balanced_plan).
    Returns (plan, fits, trials)."""
    from .costfit import (GridSpec, calibrated_dual_constraint, fit_cost_model,
                          fit_quadratic_cost_model, generate_sweep)

    reqs = list(generate_sweep(catalog).trials)
    # also measure each bucket at its memory envelope, the regime the plans actually run in
    for bucket in catalog:
        b_env = max(1, int(m_mem // bucket.seq_len))
        if (b_env, bucket.seq_len) not in reqs:
            reqs.append((b_env, bucket.seq_len))
    trials = measure_trials(runner, reqs)
    fits = {"power": fit_cost_model(trials, GridSpec(1.0, 2.4, 0.05)),
            "quadratic": fit_quadratic_cost_model(trials)}
    return fits, trials


def plan_from_fit(kind: str, model, catalog, m_mem: float):
    from .costfit import calibrated_dual_constraint, time_balanced_plan

    if kind == "power":
        return emit_plan(catalog, calibrated_dual_constraint(model, catalog, m_mem))
    return time_balanced_plan(model, catalog, m_mem)


def warm_buckets(runner: DPStepRunner, plan) -> None:
    """Run every planned (B, S) shape once on this rank (no collective) so kernels, workspaces
    and the caching allocator's blocks exist before timing; without it a rank's first encounter
    of a shape costs ~2x (allocator growth), which reads as imbalance."""
    for e in plan.entries:
        shard = RankShard(runner.rank, -1, e.bucket, e.batch_size)
        x, t, target = runner.make_batch(shard)
        with torch.autocast(runner.device.type, dtype=torch.bfloat16,
                            enabled=runner.device.type == "cuda"):
            loss = F.mse_loss(runner.block(x, t).float(), target.float())
        loss.backward()
        runner.flat_grad.zero_()
        del x, t, target, loss
    if runner.device.type == "cuda":
        torch.cuda.synchronize(runner.device)


@dataclass(frozen=True)
class RefitConfig:
    """Closed-loop recalibration (reference: cluster_sim.py:187-195, 238-241): every `every`
    steps, refit the cost model on ALL ranks' measured (B_i, S_i, T_i) so far and re-plan.
    The per-rank times are all-gathered each step, so every rank fits the same data and
    arrives at the same plan without any extra communication."""

    every: int
    m_mem: float
    cost_model: str = "quadratic"


def run_policy_steps(runner: DPStepRunner, sampler: BucketSampler, steps: int,
                     warmup: int = 0, refit: RefitConfig | None = None,
                     refit_log: list | None = None) -> list:
    from .costfit import (GridSpec, calibrated_dual_constraint, fit_cost_model,
                          fit_quadratic_cost_model, time_balanced_plan)
    from .traces import trials_from_steps

    stats, trials = [], []
    for i in range(warmup + steps):
        shards = sampler.step()
        st = runner.step(i, shards)
        if i >= warmup:
            stats.append(st)
        if refit is not None:
            trials.extend(trials_from_steps([st])[0])
            if (i + 1) % refit.every == 0 and len({(t.batch, t.seq_len) for t in trials}) >= 3:
                try:
                    if refit.cost_model == "power":
                        model = fit_cost_model(trials, GridSpec(1.0, 2.4, 0.05))
                        plan = emit_plan(sampler.catalog,
                                         calibrated_dual_constraint(model, sampler.catalog,
                                                                    refit.m_mem))
                    else:
                        model = fit_quadratic_cost_model(trials)
                        plan = time_balanced_plan(model, sampler.catalog, refit.m_mem)
                except AdaptiveLoadError as exc:  # keep the current plan (same on every rank)
                    if refit_log is not None:
                        refit_log.append({"step": i, "error": type(exc).__name__})
                    continue
                sampler.set_plan(plan)
                warm_buckets(runner, plan)
                if refit_log is not None:
                    refit_log.append({"step": i, "model": model.__dict__,
                                      "plan": plan.batch_sizes()})
    return stats


def summarize(stats: list, world: int) -> dict:
    from .costfit import analyze_bottleneck

    tok = sum(s.tokens for s in stats)
    t = sum(s.t_step_ms for s in stats) / 1e3
    bn = analyze_bottleneck(stats) if stats else None  # measured wait_sync per rank
    per_bucket = {}
    for st in stats:
        for sh, ti in zip(st.shards, st.t_compute_ms):
            per_bucket.setdefault(f"{sh.batch_size}x{sh.seq_len}", []).append(ti)
    return {
        "measured_ms_by_bucket": {k: round(float(np.mean(v)), 3) for k, v in
                                  sorted(per_bucket.items(), key=lambda kv: int(kv[0].split("x")[1]))},
        "per_step": [{"seq": [sh.seq_len for sh in st.shards],
                      "t_ms": [round(x, 2) for x in st.t_compute_ms],
                      "step_ms": round(st.t_step_ms, 2)} for st in stats],
        "steps": len(stats),
        "tokens_per_sec": tok / t if t > 0 else 0.0,
        "mean_step_ms": 1e3 * t / max(len(stats), 1),
        "mean_cv_step_measured": float(np.mean([s.cv_step for s in stats])) if world > 1 else 0.0,
        "mean_compute_cv": float(np.mean([s.compute_cv for s in stats])) if world > 1 else 0.0,
        "mean_wait_sync_ms": float(np.mean([np.mean(s.wait_sync_ms) for s in stats])),
        # reference costfit.analyze_bottleneck on the measured waits: mean wait per rank (ms)
        # and the share of steps each rank was the straggler
        "bottleneck": None if bn is None else {
            "mean_wait_ms": [round(1e3 * v, 3) for v in bn.mean_wait],
            "straggler_fraction": [round(v, 4) for v in bn.straggler_fraction]},
    }


# ------------------------------------------------------------------------------ bench entry
ARMS = ("equal_token", "dual_reference", "dual_power_fit", "dual_quadratic")
ARM_DOC = {
    "equal_token": "TokenBudget(M_mem): B = floor(M_mem / S) (scheduler.py:95-98)",
    "dual_reference": "the reference's DualConstraint(M_mem, 3e9 * (M_mem / 480k)^2, p = 2) "
                      "(cluster_sim.py:332-336): plan [300, 100, 32, 5, 1, 1] at 480k",
    "dual_power_fit": "the reference fitter on B200 trials: T = a + b B S^p grid-searched "
                      "(costfit.py:116-140), M_comp from the fit (calibrated_dual_constraint)",
    "dual_quadratic": "B200 two-term fit T = a + c1 B S + c2 B S^2, every bucket capped at the "
                      "longest bucket's B = 1 time (costfit.time_balanced_plan)",
}


def run_arms(world: int, rank: int, local: int, steps: int, warmup: int, seed: int = 42,
             token_budget: int = 480_000, m_comp: float = 0.0, arms=ARMS,
             detail: bool = True, keep_stats: bool = False) -> dict:
    """The DP step under each bucket plan in `arms`, same seed (same bucket draws) for all,
    on this process group.  Plans that need a cost model use rank 0's calibration sweep of the
    block on this GPU, broadcast so every rank builds the same plan."""
    from .catalogs import reference_default_catalog
    from .costfit import CostModel, QuadraticCostModel
    from .scheduler import DualConstraint, TokenBudget

    dev = torch.device("cuda", local)
    catalog, weights, tb, dc = reference_default_catalog()
    m_mem = token_budget
    # a different token budget scales M_comp to keep the reference's M_comp / M_mem^2
    m_comp = m_comp or dc.m_comp * (m_mem / dc.m_mem) ** 2
    plans = {"equal_token": emit_plan(catalog, TokenBudget(m_mem)),
             "dual_reference": emit_plan(catalog, DualConstraint(float(m_mem), m_comp, 2.0))}
    calib = None
    if any(a in ("dual_power_fit", "dual_quadratic") for a in arms):
        vec = torch.zeros(8, dtype=torch.float64, device=dev)
        trials = []
        if rank == 0:
            torch.manual_seed(0)
            cal_runner = DPStepRunner(WanStyleBlock(), dev, 1, 0, seed=seed)
            fits, trials = calibrate_plan(cal_runner, catalog, m_mem)
            pw, qd = fits["power"], fits["quadratic"]
            vec = torch.tensor([pw.a, pw.b, pw.p, pw.r2, qd.a, qd.c1, qd.c2, qd.r2],
                               dtype=torch.float64, device=dev)
            del cal_runner
            torch.cuda.empty_cache()
        if world > 1:
            import torch.distributed as dist

            dist.broadcast(vec, 0)
        v = [float(a) for a in vec.cpu()]
        fits = {"power": CostModel(*v[:4]), "quadratic": QuadraticCostModel(*v[4:])}
        plans["dual_power_fit"] = plan_from_fit("power", fits["power"], catalog, m_mem)
        plans["dual_quadratic"] = plan_from_fit("quadratic", fits["quadratic"], catalog, m_mem)
        calib = {"power_fit": fits["power"].__dict__, "quadratic_fit": fits["quadratic"].__dict__,
                 "trials": [[t.batch, t.seq_len, round(t.step_time, 6)] for t in trials],
                 "predicted_ms": {k: [round(1e3 * fits[k].predict(e.batch_size, e.bucket.seq_len), 3)
                                      for e in plans[f"dual_{'power_fit' if k == 'power' else k}"].entries]
                                  for k in ("power", "quadratic")}}
    out, all_stats = {}, {}
    for name in arms:
        plan = plans[name]
        torch.manual_seed(0)
        runner = DPStepRunner(WanStyleBlock(), dev, world, rank, seed=seed)
        sampler = BucketSampler(catalog, weights, plan, max(world, 1), seed)
        warm_buckets(runner, plan)
        stats = run_policy_steps(runner, sampler, steps, warmup=warmup)
        out[name] = summarize(stats, world)
        out[name]["plan"] = plan.batch_sizes()
        if not detail:
            out[name].pop("per_step", None)
        if keep_stats:
            all_stats[name] = stats
        del runner
        torch.cuda.empty_cache()
    base = out.get("equal_token")
    res = {
        "config": {"workload": "Wan-2.1-1.3B-style block (D=1536, 12 heads, FFN 8960), fused "
                               "AdaLN x2, reference default catalog, per-rank draws",
                   "token_budget": m_mem, "m_comp_reference": m_comp,
                   "arms": {a: ARM_DOC[a] for a in arms},
                   "plans": {a: plans[a].batch_sizes() for a in arms},
                   "parallelism": f"dp{world}, one NCCL all-reduce per step", "steps": steps,
                   "seed": seed},
        "policies": out,
        "calibration": calib,
        "imbalance": {a: {"compute_cv_pct": out[a]["mean_compute_cv"],
                          "cv_step_measured": out[a]["mean_cv_step_measured"],
                          "wait_sync_ms": out[a]["mean_wait_sync_ms"],
                          "tokens_per_sec": out[a]["tokens_per_sec"],
                          "throughput_vs_equal_token": (None if base is None else
                                                        out[a]["tokens_per_sec"]
                                                        / max(base["tokens_per_sec"], 1e-9) - 1.0)}
                      for a in arms},
    }
    if keep_stats:
        res["_stats"] = all_stats
        res["_plans"] = {a: plans[a] for a in arms}
    return res


def run_ab(world: int, rank: int, local: int, steps: int, warmup: int, seed: int = 42,
           token_budget: int = 480_000, m_comp: float = 0.0, plan_kind: str = "calibrated",
           cost_model: str = "quadratic", detail: bool = True) -> dict:
    """Two-arm form (equal token vs one dual plan) kept for the earlier tools: the dual arm is
    the calibrated plan of `cost_model` or, with plan_kind="reference", the reference's."""
    dual = ("dual_reference" if plan_kind == "reference" else
            "dual_power_fit" if cost_model == "power" else "dual_quadratic")
    r = run_arms(world, rank, local, steps, warmup, seed, token_budget, m_comp,
                 ("equal_token", dual), detail)
    pol = {"equal_token": r["policies"]["equal_token"], "dual": r["policies"][dual]}
    r["policies"] = pol
    r["config"]["plan_equal_token"] = pol["equal_token"]["plan"]
    r["config"]["plan_dual"] = pol["dual"]["plan"]
    r["imbalance"] = {
        "compute_cv_equal_token_pct": pol["equal_token"]["mean_compute_cv"],
        "compute_cv_dual_pct": pol["dual"]["mean_compute_cv"],
        "cv_step_measured_equal_token": pol["equal_token"]["mean_cv_step_measured"],
        "cv_step_measured_dual": pol["dual"]["mean_cv_step_measured"],
        "wait_sync_ms_equal_token": pol["equal_token"]["mean_wait_sync_ms"],
        "wait_sync_ms_dual": pol["dual"]["mean_wait_sync_ms"],
    }
    r["throughput_gain_vs_equal_token"] = (pol["dual"]["tokens_per_sec"]
                                           / max(pol["equal_token"]["tokens_per_sec"], 1e-9) - 1.0)
    if r.get("calibration"):
        key = "power" if dual == "dual_power_fit" else "quadratic"
        r["calibration"]["cost_model"] = key
        r["calibration"]["predicted_ms"] = r["calibration"]["predicted_ms"].get(key)
    return r


def write_traces(trace_dir, res: dict, world: int, command: str) -> dict:
    """The measured steps in the reference's file formats, one set per arm:
    trial trace JSONL (B_i, S_i, T_i per rank and step -- what the reference CLI's `fit`
    consumes) with a manifest sidecar, plan JSON, the fitted models, per-step metrics CSV
    (t_sync, cv_step, compute_cv, tokens/s, theta) and a summary JSON, all with manifests."""
    from pathlib import Path

    from .costfit import CostModel
    from .manifest import make_manifest
    from .sampler import latent_units
    from .shapes import LatentGeometry
    from .traces import (save_metrics_csv, save_model, save_plan, save_summary, save_trace,
                         trials_from_steps, write_manifest_sidecar)

    d = Path(trace_dir)
    d.mkdir(parents=True, exist_ok=True)
    cfg = res["config"]
    written, rows = {}, {}
    geom = LatentGeometry()
    for arm, stats in res["_stats"].items():
        trials, workers = trials_from_steps(stats)
        tr = d / f"trace_{arm}.jsonl"
        save_trace(tr, trials, workers)
        man = make_manifest(command, {**cfg, "arm": arm}, [], [tr.name], cfg["seed"])
        write_manifest_sidecar(tr, man)
        pl = d / f"plan_{arm}.json"
        save_plan(pl, res["_plans"][arm], make_manifest(command, {**cfg, "arm": arm}, [],
                                                         [pl.name], cfg["seed"]))
        rows[arm] = []
        for st in stats:
            t_sync = max(st.t_compute_ms) / 1e3
            units = sum(latent_units(sh, geom) for sh in st.shards)
            rows[arm].append({"t_sync": t_sync, "cv_step": st.cv_step,
                              "compute_cv": st.compute_cv, "tokens_per_sec": st.tokens / t_sync,
                              "theta": units / t_sync})
        written[arm] = [tr.name, tr.name + ".manifest.json", pl.name]
    mc = d / "metrics.csv"
    save_metrics_csv(mc, rows)
    write_manifest_sidecar(mc, make_manifest(command, cfg, [], [mc.name], cfg["seed"]))
    if res.get("calibration"):
        pf = res["calibration"]["power_fit"]
        save_model(d / "model_power_fit.json", CostModel(pf["a"], pf["b"], pf["p"], pf["r2"]),
                   make_manifest(command, cfg, [], ["model_power_fit.json"], cfg["seed"]))
    summ = {k: v for k, v in res.items() if not k.startswith("_")}
    for pol in summ["policies"].values():
        pol.pop("per_step", None)
    save_summary(d / "summary.json", {"world": world, **summ},
                 make_manifest(command, cfg, [], ["summary.json"], cfg["seed"]))
    return {"dir": str(d), "files": sorted(p.name for p in d.iterdir())}


def bench_main(args, rest, world: int, rank: int, local: int) -> None:
    """``bench.py --workload dit``: tokens/s of the DiT-block DP step at N GPUs under each bucket
    plan (ARMS: equal token, the reference's dual constraint, the reference fitter's power-law
    dual on B200 trials, the two-term time-balanced plan), same draws for every arm, with the
    measured per-rank imbalance.  ``value`` is the time-balanced arm's tokens/s.
    ``--trace-dir DIR`` writes the measured steps in the reference's file formats."""
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--policy-steps", type=int, default=0)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--token-budget", type=int, default=480_000)
    ap.add_argument("--m-comp", type=float, default=0.0)
    ap.add_argument("--arms", default=",".join(ARMS))
    ap.add_argument("--trace-dir", default="")
    extra = ap.parse_args(rest)
    steps = extra.policy_steps or args.steps
    arms = tuple(a for a in extra.arms.split(",") if a)
    bad = [a for a in arms if a not in ARMS]
    if bad:
        raise SystemExit(f"unknown arm(s) {bad}; choose from {ARMS}")
    res = run_arms(world, rank, local, steps, args.warmup, extra.seed, extra.token_budget,
                   extra.m_comp, arms, detail=True, keep_stats=bool(extra.trace_dir))
    if rank == 0:
        head = "dual_quadratic" if "dual_quadratic" in arms else arms[-1]
        pol = res["policies"][head]
        if extra.trace_dir:
            res["traces"] = write_traces(extra.trace_dir, res, world,
                                         f"bench.py --workload dit --gpus {world}")
        line = {
            "metric": "DiT-block DP step tokens/s (dual-constraint buckets)",
            "value": round(pol["tokens_per_sec"], 1), "unit": "tokens/s", "arm": head,
            "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "ms_per_step": round(pol["mean_step_ms"], 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            **{k: v for k, v in res.items() if not k.startswith("_")},
        }
        print(json.dumps(line), flush=True)
