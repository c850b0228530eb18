"""Per-rank bucket sampler feeding the data-parallel step, and the imbalance metrics.

Reference: cluster_sim.py:113-131 (sample_assignments), :134-158 (simulate_step), :161-174
(cv_step, compute_cv), :198-300 (run_policy / run_experiment).

Every step draws ONE global vector of bucket indices from a seeded ``numpy.random.Generator``
(PCG64), identical on every rank, and rank i takes entry i -- so assignment needs no
communication and is bit-identical to the reference's ``sample_assignments`` for the same
generator state.  The draw is the inverse-CDF form of ``Generator.choice(n, size, p=w)``:
``cdf = cumsum(w); cdf /= cdf[-1]; idx = searchsorted(cdf, rng.random(size), 'right')``,
consuming one uniform double per rank, exactly as numpy's ``choice`` does.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import AllZero, PlanMismatch, ZeroMean
from .scheduler import BucketPlan, physical_load
from .shapes import Bucket, LatentGeometry, visual_tokens

__all__ = ["RankShard", "BucketSampler", "sample_assignments", "draw_indices", "cv_step",
           "compute_cv", "PolicyMetrics", "simulate_policy", "compare_policies", "NOISE_FLOOR",
           "CostParams"]

NOISE_FLOOR = 0.01  # cluster_sim.py:42


def _validated_cdf(weights, n_buckets: int) -> np.ndarray:
    w = np.asarray(weights, dtype=np.float64)
    if w.shape != (n_buckets,):
        raise PlanMismatch("one weight per bucket required")
    if abs(float(w.sum()) - 1.0) > 1e-9:
        raise ValueError(f"weights must sum to 1, got {w.sum()}")
    if (w < 0).any():
        raise ValueError("weights must be non-negative")
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    return cdf


def draw_indices(cdf: np.ndarray, num_workers: int, rng: np.random.Generator) -> np.ndarray:
    """One bucket index per worker: inverse CDF of one uniform double each."""
    u = rng.random(num_workers)
    return np.searchsorted(cdf, u, side="right").astype(np.int64)


def _planned(plan: BucketPlan, catalog) -> list[int]:
    by_shape = {e.bucket.shape: e.batch_size for e in plan.entries}
    missing = [b.shape for b in catalog if b.shape not in by_shape]
    if missing:
        raise PlanMismatch(f"plan does not cover shape {missing[0]}")
    return [by_shape[b.shape] for b in catalog]


def sample_assignments(catalog, weights, plan: BucketPlan, num_workers: int,
                       rng: np.random.Generator) -> list[tuple[Bucket, int]]:
    """Independent weighted bucket draw per worker; batch size from the plan (cluster_sim.py:113)."""
    cdf = _validated_cdf(weights, len(catalog))
    batches = _planned(plan, catalog)
    idx = draw_indices(cdf, num_workers, rng)
    return [(catalog[i], batches[i]) for i in idx]


@dataclass(frozen=True)
class RankShard:
    """What one data-parallel rank processes in one step: B samples of one bucket."""

    rank: int
    bucket_index: int
    bucket: Bucket
    batch_size: int

    @property
    def seq_len(self) -> int:
        return self.bucket.seq_len

    @property
    def tokens(self) -> int:
        return self.batch_size * self.bucket.seq_len

    @property
    def load(self) -> int:
        return physical_load(self.batch_size, self.bucket.seq_len)


class BucketSampler:
    """Step-synchronous sampler: every rank constructs it with the same seed and calls ``step``.

    ``noise_draws`` > 0 additionally consumes that many standard normals per step after the
    bucket draw -- the simulator's jitter draw (cluster_sim.py:141) -- so the index stream can
    be replayed against the reference's ``run_policy`` (used by the parity tests and by
    ``compare_policies``); the training step leaves it at 0.
    """

    def __init__(self, catalog, weights, plan: BucketPlan, world_size: int,
                 rng: np.random.Generator | int = 0, noise_draws: int = 0,
                 noise_sigma: float = 0.0):
        self.catalog = list(catalog)
        self.cdf = _validated_cdf(weights, len(self.catalog))
        self.batches = _planned(plan, self.catalog)
        self.world_size = int(world_size)
        self.rng = rng if isinstance(rng, np.random.Generator) else np.random.default_rng(rng)
        self.noise_draws = noise_draws
        self.noise_sigma = noise_sigma
        self.last_noise = None

    def set_plan(self, plan: BucketPlan) -> None:
        """Swap the per-bucket batch sizes (closed-loop refit); the draw stream is unaffected."""
        self.batches = _planned(plan, self.catalog)

    def step(self) -> list[RankShard]:
        idx = draw_indices(self.cdf, self.world_size, self.rng)
        if self.noise_draws:
            self.last_noise = self.rng.normal(0.0, self.noise_sigma, self.noise_draws)
        return [RankShard(r, int(i), self.catalog[i], self.batches[i]) for r, i in enumerate(idx)]


# ------------------------------------------------------------------------------- metrics
def cv_step(values) -> float:
    """Range-ratio imbalance (max - min) / max (cluster_sim.py:161-166)."""
    v = np.asarray(values, dtype=np.float64)
    if v.size == 0 or float(v.max()) <= 0.0:
        raise AllZero("range-ratio CV needs a positive maximum")
    hi = v.max()
    return float((hi - v.min()) / hi)


def compute_cv(loads) -> float:
    """100 * population std / mean of per-rank loads (cluster_sim.py:169-174)."""
    v = np.asarray(loads, dtype=np.float64)
    if v.size == 0 or float(v.mean()) == 0.0:
        raise ZeroMean("std/mean CV needs a nonzero mean")
    return float(100.0 * v.std() / v.mean())


# ------------------------------------------------------------------ simulated policy A/B
@dataclass(frozen=True)
class CostParams:
    """Simulator ground-truth cost T = a + b * B * S^p (cluster_sim.py:45-49)."""

    a: float = 2.0
    b: float = 1e-9
    p: float = 2.0


@dataclass(frozen=True)
class PolicyMetrics:
    mean_compute_cv: float        # 100 * std/mean of B*S^2 over ranks, averaged over steps
    mean_compute_cv_range: float  # (max-min)/max of B*S^2
    mean_cv_step: float           # (max-min)/max of simulated step times
    mean_time_cv_stdmean: float
    mean_t_sync: float
    tokens_per_sec: float         # total tokens / total synchronized time
    steps: int
    rows: tuple = ()              # per-step metrics (traces.METRICS_COLUMNS) when requested


def simulate_policy(catalog, weights, plan: BucketPlan, world_size: int, steps: int,
                    rng: np.random.Generator, cost: CostParams = CostParams(),
                    noise_sigma: float = 0.03, geom: LatentGeometry | None = None,
                    keep_rows: bool = False) -> PolicyMetrics:
    """The reference's run_policy metrics without refit (cluster_sim.py:198-246).

    Consumes the generator exactly like the reference (N uniforms for the draw, then N normals
    for the jitter each step), so compute_cv per step is bit-identical to it.
    """
    sampler = BucketSampler(catalog, weights, plan, world_size, rng, noise_draws=world_size,
                            noise_sigma=noise_sigma)
    geom = geom or LatentGeometry()
    ccv, ccr, cvs, tcv, tsync, toks, rows = [], [], [], [], [], [], []
    for _ in range(steps):
        shards = sampler.step()
        noise = np.maximum(NOISE_FLOOR, 1.0 + sampler.last_noise)
        times = [(cost.a + cost.b * sh.batch_size * float(sh.seq_len) ** cost.p) * float(nz)
                 for sh, nz in zip(shards, noise)]
        loads = [sh.load for sh in shards]
        ccv.append(compute_cv(loads))
        ccr.append(cv_step(loads))
        cvs.append(cv_step(times))
        tcv.append(compute_cv(times))
        tsync.append(max(times))
        toks.append(sum(sh.tokens for sh in shards))
        if keep_rows:
            units = sum(latent_units(sh, geom) for sh in shards)
            rows.append({"t_sync": tsync[-1], "cv_step": cvs[-1], "compute_cv": ccv[-1],
                         "tokens_per_sec": toks[-1] / tsync[-1], "theta": units / tsync[-1]})
    t = np.asarray(tsync)
    return PolicyMetrics(float(np.mean(ccv)), float(np.mean(ccr)), float(np.mean(cvs)),
                         float(np.mean(tcv)), float(t.mean()), float(np.sum(toks) / t.sum()),
                         steps, tuple(rows))


def compare_policies(catalog, weights, plan_baseline: BucketPlan, plan_dual: BucketPlan,
                     world_size: int, steps: int = 500, seed: int = 42,
                     cost: CostParams = CostParams(), noise_sigma: float = 0.03) -> dict:
    """Equal-token vs dual-constraint A/B with the reference's stream split (cluster_sim.py:258-300)."""
    child_a, child_b = np.random.SeedSequence(seed).spawn(2)
    a = simulate_policy(catalog, weights, plan_baseline, world_size, steps,
                        np.random.default_rng(child_a), cost, noise_sigma)
    b = simulate_policy(catalog, weights, plan_dual, world_size, steps,
                        np.random.default_rng(child_b), cost, noise_sigma)
    strip = lambda m: {k: v for k, v in m.__dict__.items() if k != "rows"}  # noqa: E731
    return {
        "equal_token": strip(a), "dual": strip(b),
        "compute_cv_reduction": (a.mean_compute_cv - b.mean_compute_cv) / a.mean_compute_cv,
        "tokens_per_sec_gain": b.tokens_per_sec / a.tokens_per_sec - 1.0,
    }


def latent_units(shard: RankShard, geom: LatentGeometry) -> int:
    """Theta numerator: batch x visual tokens (cluster_sim.py:177-184, 224-226)."""
    return shard.batch_size * visual_tokens(shard.bucket.shape, geom)
