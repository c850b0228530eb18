"""Trace, plan, model and metrics files in the reference's schemas (reference: io.py:99-203).

SURVEY 8(f) rank 3: the B200 DP step emits its per-rank measurements in the same text formats
the reference CLI reads (`fit` consumes trial JSONL, `simulate`/`plan` consume plan and model
JSON, metrics go to CSV), so the reference tooling can fit, plan and compare on real B200
traces.  Deterministic text: sorted keys, 2-space JSON indent, `repr` floats in CSV.
"""

from __future__ import annotations

import csv
import json
from pathlib import Path

from dataclasses import dataclass

from .costfit import CostModel, Trial
from .manifest import RunManifest
from .scheduler import Binding, BucketPlan, PlanEntry
from .shapes import Bucket, LatentGeometry, MediaShape, build_catalog

__all__ = ["save_trace", "load_trace", "save_plan", "load_plan", "save_model", "load_model",
           "save_metrics_csv", "METRICS_COLUMNS", "trials_from_steps", "load_catalog",
           "save_catalog", "ClusterCost", "ClusterConfig", "load_cluster_config", "save_summary",
           "write_manifest_sidecar"]

METRICS_COLUMNS = ["step", "policy", "t_sync", "cv_step", "compute_cv", "tokens_per_sec", "theta"]


def _write_json(path, doc) -> None:
    Path(path).write_text(json.dumps(doc, sort_keys=True, indent=2) + "\n")


def _manifest_doc(manifest) -> dict:
    if manifest is None:
        return {}
    return manifest.to_dict() if isinstance(manifest, RunManifest) else dict(manifest)


def write_manifest_sidecar(path, manifest) -> None:
    """Manifest of a line/row-oriented artifact (JSONL, CSV) in ``<path>.manifest.json``."""
    _write_json(str(path) + ".manifest.json", _manifest_doc(manifest))


# ------------------------------------------------------------------ catalogs (io.py:32-80)
_GEOM_DEFAULTS = {"temporal_factor": 8, "width_factor": 16, "height_factor": 16, "text_tokens": 0}


def load_catalog(path):
    """(buckets, weights, geometry) from a catalog JSON: either a list of
    {frames, height, width, count} or {"shapes": [...], "geometry": {...}} (missing geometry
    keys take the reference defaults); weights are the normalised sample counts."""
    doc = json.loads(Path(path).read_text())
    shapes, geom_doc = (doc, {}) if isinstance(doc, list) else (doc["shapes"], doc.get("geometry", {}))
    g = {k: geom_doc.get(k, v) for k, v in _GEOM_DEFAULTS.items()}
    geom = LatentGeometry(temporal_factor=g["temporal_factor"], width_factor=g["width_factor"],
                          height_factor=g["height_factor"], text_tokens=g["text_tokens"])
    catalog = build_catalog([(MediaShape(r["frames"], r["height"], r["width"]), r["count"])
                             for r in shapes], geom)
    n = sum(b.sample_count for b in catalog)
    return catalog, [b.sample_count / n for b in catalog], geom


def save_catalog(path, catalog, geom: LatentGeometry) -> None:
    _write_json(path, {
        "shapes": [{"frames": b.shape.frames, "height": b.shape.height, "width": b.shape.width,
                    "count": b.sample_count} for b in catalog],
        "geometry": {k: getattr(geom, k) for k in _GEOM_DEFAULTS}})


# ------------------------------------------------------------ cluster config (io.py:83-96)
@dataclass(frozen=True)
class ClusterCost:
    a: float = 2.0
    b: float = 1e-9
    p: float = 2.0


@dataclass(frozen=True)
class ClusterConfig:
    """The reference simulator's cluster description (cluster_sim.py:53-63); on B200 the DP
    step takes its world size from torch.distributed and measures the per-rank cost, so only
    num_workers / seed / steps steer a run, the cost block is carried for the reference tools."""

    num_workers: int = 16
    cost: ClusterCost = ClusterCost()
    noise_sigma: float = 0.03
    seed: int = 42
    steps: int = 500


def load_cluster_config(path, seed_override: int | None = None) -> ClusterConfig:
    doc = json.loads(Path(path).read_text())
    c = doc.get("cost", {})
    d = ClusterConfig()
    return ClusterConfig(
        num_workers=doc.get("num_workers", d.num_workers),
        cost=ClusterCost(c.get("a", d.cost.a), c.get("b", d.cost.b), c.get("p", d.cost.p)),
        noise_sigma=doc.get("noise_sigma", d.noise_sigma),
        seed=doc.get("seed", d.seed) if seed_override is None else seed_override,
        steps=doc.get("steps", d.steps))


def save_summary(path, summary: dict, manifest=None) -> None:
    _write_json(path, {**summary, "manifest": _manifest_doc(manifest)})


def save_trace(path, trials, workers=None) -> None:
    """One JSON object per line: batch, seq_len, step_time_sync (s) [, worker] (io.py:158-165)."""
    lines = []
    for i, t in enumerate(trials):
        row = {"batch": t.batch, "seq_len": t.seq_len, "step_time_sync": t.step_time}
        if workers is not None:
            row["worker"] = workers[i]
        lines.append(json.dumps(row, sort_keys=True))
    Path(path).write_text("".join(line + "\n" for line in lines))


def load_trace(path) -> list:
    out = []
    for line in Path(path).read_text().splitlines():
        if line.strip():
            r = json.loads(line)
            out.append(Trial(r["batch"], r["seq_len"], r["step_time_sync"]))
    return out


def save_plan(path, plan: BucketPlan, manifest=None) -> None:
    entries = [{"frames": e.bucket.shape.frames, "height": e.bucket.shape.height,
                "width": e.bucket.shape.width, "seq_len": e.bucket.seq_len,
                "sample_count": e.bucket.sample_count, "batch_size": e.batch_size,
                "binding": None if e.binding is None else e.binding.value}
               for e in plan.entries]
    _write_json(path, {"entries": entries, "manifest": _manifest_doc(manifest)})


def load_plan(path) -> BucketPlan:
    doc = json.loads(Path(path).read_text())
    return BucketPlan(tuple(
        PlanEntry(Bucket(MediaShape(e["frames"], e["height"], e["width"]), e["seq_len"],
                         e["sample_count"]), e["batch_size"],
                  None if e["binding"] is None else Binding(e["binding"]))
        for e in doc["entries"]))


def save_model(path, model: CostModel, manifest=None) -> None:
    _write_json(path, {"a": model.a, "b": model.b, "p": model.p, "r2": model.r2,
                       "manifest": _manifest_doc(manifest)})


def load_model(path) -> CostModel:
    doc = json.loads(Path(path).read_text())
    return CostModel(doc["a"], doc["b"], doc["p"], doc["r2"])


def save_metrics_csv(path, rows_by_policy: dict) -> None:
    """rows_by_policy: policy -> list of dicts with the METRICS_COLUMNS fields (per step)."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(METRICS_COLUMNS)
        for policy, rows in rows_by_policy.items():
            for i, r in enumerate(rows):
                w.writerow([i, policy] + [repr(float(r[c])) for c in METRICS_COLUMNS[2:]])


def trials_from_steps(stats) -> tuple[list, list]:
    """Per-rank (B_i, S_i, T_i) of measured DP steps as reference Trials (seconds) + worker ids."""
    trials, workers = [], []
    for st in stats:
        for rank, (sh, t_ms) in enumerate(zip(st.shards, st.t_compute_ms)):
            trials.append(Trial(sh.batch_size, sh.seq_len, t_ms / 1e3))
            workers.append(rank)
    return trials, workers
