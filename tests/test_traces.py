"""Trace / plan / model / metrics files are byte-identical to the reference's writers
(tests/golden/io/ was written by the reference's io.py -- make_golden.py:make_io)."""

import json
from pathlib import Path

import numpy as np

from paper_2605_17923_b200 import traces
from paper_2605_17923_b200.catalogs import reference_default_catalog
from paper_2605_17923_b200.costfit import Trial, fit_cost_model
from paper_2605_17923_b200.sampler import simulate_policy
from paper_2605_17923_b200.scheduler import emit_plan

IO = Path(__file__).resolve().parent / "golden" / "io"


def test_plan_files_identical(tmp_path):
    cat, w, tb, dc = reference_default_catalog()
    for name, pol in (("plan_dual.json", dc), ("plan_equal_token.json", tb)):
        ref = (IO / name).read_text()
        man = json.loads(ref)["manifest"]
        traces.save_plan(tmp_path / name, emit_plan(cat, pol), man)
        assert (tmp_path / name).read_text() == ref
        plan = traces.load_plan(IO / name)
        assert plan.batch_sizes() == emit_plan(cat, pol).batch_sizes()


def test_trace_and_model_files_identical(tmp_path):
    trials = [Trial(b, s, 2.0 + 1e-9 * b * s ** 2) for b, s in ((1, 1600), (3, 24000), (1, 52800))]
    traces.save_trace(tmp_path / "trace.jsonl", trials, workers=[0, 1, 0])
    assert (tmp_path / "trace.jsonl").read_text() == (IO / "trace.jsonl").read_text()
    assert traces.load_trace(IO / "trace.jsonl") == trials
    ref = (IO / "model.json").read_text()
    traces.save_model(tmp_path / "model.json", fit_cost_model(trials), json.loads(ref)["manifest"])
    assert (tmp_path / "model.json").read_text() == ref


def test_metrics_csv_identical(tmp_path):
    cat, w, tb, dc = reference_default_catalog()
    ss = np.random.SeedSequence(42)
    ca, cb = ss.spawn(2)
    rows = {}
    for name, pol, child in (("equal_token", tb, ca), ("dual", dc, cb)):
        m = simulate_policy(cat, w, emit_plan(cat, pol), 4, 5, np.random.default_rng(child),
                            keep_rows=True)
        rows[name] = list(m.rows)
    traces.save_metrics_csv(tmp_path / "metrics.csv", rows)
    assert (tmp_path / "metrics.csv").read_text() == (IO / "metrics.csv").read_text()
