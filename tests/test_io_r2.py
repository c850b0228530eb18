"""Catalog / cluster-config / summary / manifest formats, config digests and the bottleneck
analysis against files and values the REFERENCE wrote (tests/golden/io/, make_golden.py
make_io_r2), plus the ``adaptiveload`` drop-in import path."""

import json
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

from paper_2605_17923_b200 import traces
from paper_2605_17923_b200.catalogs import reference_default_catalog
from paper_2605_17923_b200.costfit import CostModel, analyze_bottleneck
from paper_2605_17923_b200.errors import EmptyRecords
from paper_2605_17923_b200.manifest import RunManifest, config_digest, make_manifest
from paper_2605_17923_b200.shapes import LatentGeometry, MediaShape, build_catalog

IO = Path(__file__).resolve().parent / "golden" / "io"
G = json.loads((IO / "io_r2.json").read_text())


def test_save_catalog_identical(tmp_path):
    cat, _, _, _ = reference_default_catalog()
    traces.save_catalog(tmp_path / "c.json", cat, LatentGeometry())
    assert (tmp_path / "c.json").read_text() == (IO / "catalog_default.json").read_text()
    geom4 = LatentGeometry(temporal_factor=4, width_factor=16, height_factor=16, text_tokens=0)
    wan = build_catalog([(MediaShape(1, 480, 832), 40), (MediaShape(81, 480, 832), 4),
                         (MediaShape(81, 720, 1280), 2)], geom4)
    traces.save_catalog(tmp_path / "w.json", wan, geom4)
    assert (tmp_path / "w.json").read_text() == (IO / "catalog_wan_l4.json").read_text()


@pytest.mark.parametrize("name", ["catalog_default.json", "catalog_wan_l4.json", "catalog_list.json"])
def test_load_catalog_matches_reference(name):
    cat, w, g = traces.load_catalog(IO / name)
    ref = G["loaded_catalogs"][name]
    assert [b.seq_len for b in cat] == ref["seq"]
    assert [b.sample_count for b in cat] == ref["count"]
    assert w == ref["weights"]
    assert [g.temporal_factor, g.width_factor, g.height_factor, g.text_tokens] == ref["geometry"]


def test_load_cluster_config_matches_reference():
    for key, ref in G["clusters"].items():
        name, seed = key.split(":")
        c = traces.load_cluster_config(IO / name, None if seed == "None" else int(seed))
        assert [c.num_workers, c.cost.a, c.cost.b, c.cost.p, c.noise_sigma, c.seed,
                c.steps] == ref, key


def test_summary_and_sidecar_identical(tmp_path):
    ref = json.loads((IO / "summary.json").read_text())
    man = RunManifest.from_dict(ref["manifest"])
    traces.save_summary(tmp_path / "summary.json", {"cv_step": 0.25, "tokens_per_sec": 1234.5,
                                                     "policies": ["equal_token", "dual"]}, man)
    assert (tmp_path / "summary.json").read_text() == (IO / "summary.json").read_text()
    traces.write_manifest_sidecar(tmp_path / "trace.jsonl", man)
    assert ((tmp_path / "trace.jsonl.manifest.json").read_text()
            == (IO / "trace.jsonl.manifest.json").read_text())


def test_config_digest_matches_reference():
    for payload, digest in G["digests"]:
        assert config_digest(payload) == digest
    # key order does not matter; the manifest helper digests the resolved configuration
    assert config_digest({"a": 2, "b": 1}) == config_digest({"b": 1, "a": 2})
    m = make_manifest("plan", {"b": 1, "a": 2}, ["catalog.json"], ["plan.json"], 42)
    assert m.config_digest == config_digest({"a": 2, "b": 1}) == G["digests"][1][1]
    assert RunManifest.from_dict(m.to_dict()) == m


def _as_json(r):
    return {"mean_wait": [float(v) for v in r.mean_wait],
            "straggler_fraction": [float(v) for v in r.straggler_fraction],
            "suggested_m_comp": r.suggested_m_comp}


def test_bottleneck_analysis_matches_reference():
    waits = G["bottleneck"]["waits"]
    recs = [SimpleNamespace(per_worker=[SimpleNamespace(wait_sync=v) for v in row]) for row in waits]
    assert _as_json(analyze_bottleneck(recs)) == G["bottleneck"]["result"]
    model = CostModel(a=2.0, b=1e-9, p=2.0, r2=1.0)
    assert _as_json(analyze_bottleneck(recs, model, 62.0)) == G["bottleneck"]["result_model"]
    # the same numbers from a plain array and from B200 StepStats-like records (ms)
    assert _as_json(analyze_bottleneck(np.array(waits))) == G["bottleneck"]["result"]
    ms = [SimpleNamespace(wait_sync_ms=[v * 1e3 for v in row]) for row in waits]
    got = _as_json(analyze_bottleneck(ms))
    np.testing.assert_allclose(got["mean_wait"], G["bottleneck"]["result"]["mean_wait"], rtol=1e-12)
    assert got["straggler_fraction"] == G["bottleneck"]["result"]["straggler_fraction"]
    with pytest.raises(EmptyRecords):
        analyze_bottleneck([])


def test_adaptiveload_drop_in_import_path():
    import adaptiveload
    from adaptiveload import adaln, io, manifest, scheduler, shapes
    from adaptiveload.adaln import (AdalnGrads, AdalnOutput, MemoryMode, TileConfig,  # noqa: F401
                                    activation_bytes, adaln_backward_dtile, adaln_backward_naive,
                                    adaln_forward, gradcheck)
    from adaptiveload.cluster_sim import default_catalog, default_dual_constraint, sample_assignments  # noqa: F401
    from adaptiveload.errors import (AdaptiveLoadError, EmptyRecords as E2, InvalidTile,  # noqa: F401
                                     NonFiniteInput, ShapeMismatch, StaleStats)

    assert set(adaln.__all__) >= {"AdalnOutput", "AdalnGrads", "TileConfig", "MemoryMode",
                                  "BACKEND", "adaln_forward", "adaln_backward_naive",
                                  "adaln_backward_dtile", "activation_bytes", "gradcheck",
                                  "GradcheckReport"}
    assert adaptiveload.adaln.adaln_forward.__module__.startswith("paper_2605_17923_b200")
    assert io.load_catalog is traces.load_catalog and manifest.config_digest is config_digest
    cat, w = default_catalog()
    assert scheduler.emit_plan(cat, default_dual_constraint()).batch_sizes() == [300, 100, 32, 5, 1, 1]
    assert shapes.sequence_length(shapes.MediaShape(81, 480, 832),
                                  shapes.LatentGeometry(temporal_factor=4)) == 32760


def test_dp_step_trace_writer(tmp_path):
    """bench.py --workload dit --trace-dir: measured DP steps in the reference formats."""
    from paper_2605_17923_b200.dp_step import StepStats, summarize, write_traces
    from paper_2605_17923_b200.sampler import RankShard
    from paper_2605_17923_b200.scheduler import TokenBudget, emit_plan

    cat, w, tb, dc = reference_default_catalog()
    plan = emit_plan(cat, tb)
    stats = []
    for i in range(3):
        shards = [RankShard(r, k, cat[k], plan.entries[k].batch_size) for r, k in enumerate((0, 3))]
        t = [100.0 + 10 * i, 140.0]
        stats.append(StepStats(i, shards, t, 150.0, sum(s.tokens for s in shards),
                               [s.load for s in shards], 1 - t[0] / t[1], 50.0,
                               [max(t) - v for v in t]))
    res = {"config": {"seed": 42, "workload": "unit"}, "calibration": None,
           "policies": {"equal_token": summarize(stats, 2)},
           "_stats": {"equal_token": stats}, "_plans": {"equal_token": plan}}
    out = write_traces(tmp_path, res, 2, "unit-test")
    assert {"trace_equal_token.jsonl", "trace_equal_token.jsonl.manifest.json",
            "plan_equal_token.json", "metrics.csv", "metrics.csv.manifest.json",
            "summary.json"} <= set(out["files"])
    trials = traces.load_trace(tmp_path / "trace_equal_token.jsonl")
    assert [(t.batch, t.seq_len) for t in trials[:2]] == [(plan.entries[0].batch_size, cat[0].seq_len),
                                                         (plan.entries[3].batch_size, cat[3].seq_len)]
    assert trials[1].step_time == 0.14
    assert traces.load_plan(tmp_path / "plan_equal_token.json").batch_sizes() == plan.batch_sizes()
    head = (tmp_path / "metrics.csv").read_text().splitlines()[0]
    assert head == ",".join(traces.METRICS_COLUMNS)
    summ = json.loads((tmp_path / "summary.json").read_text())
    assert summ["policies"]["equal_token"]["bottleneck"]["straggler_fraction"] == [0.0, 1.0]
    assert len(summ["manifest"]["config_digest"]) == 64
