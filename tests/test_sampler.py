"""Sampler path (shapes -> batch rule -> per-rank draws -> imbalance metrics) vs the reference.

Golden values in tests/golden/sampler_golden.json were produced by the reference itself
(tests/golden/make_golden.py).  Bucket assignment must be BIT-EXACT (north_star).
"""

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import sampler_oracle as so
from paper_2605_17923_b200.catalogs import reference_default_catalog, wan21_catalog
from paper_2605_17923_b200.errors import AllZero, EmptyCatalog, PlanMismatch, ZeroMean
from paper_2605_17923_b200.sampler import (
    BucketSampler, compare_policies, compute_cv, cv_step, sample_assignments)
from paper_2605_17923_b200.scheduler import (
    Binding, DualConstraint, TokenBudget, dual_constraint_batch, emit_plan, equal_token_batch,
    physical_load)
from paper_2605_17923_b200.shapes import (
    Bucket, LatentGeometry, MediaShape, WAN21_GEOMETRY, build_catalog, sequence_length)


def _catalog(name):
    if name == "default":
        cat, w, tb, dc = reference_default_catalog()
    else:
        cat, w, tb, dc = wan21_catalog()
    return cat, w, tb, dc


# ------------------------------------------------------------------ batch rule
def test_dual_constraint_batch_matches_reference(sampler_golden):
    for s, m_mem, m_comp, p, b, binding in sampler_golden["dual_constraint_batch"]:
        got_b, got_binding = dual_constraint_batch(s, DualConstraint(m_mem, m_comp, p))
        assert (got_b, got_binding.value) == (b, binding), (s, m_mem, m_comp, p)


def test_equal_token_batch_matches_reference(sampler_golden):
    for s, t, b in sampler_golden["equal_token_batch"]:
        assert equal_token_batch(s, TokenBudget(t)) == b


def test_batch_rule_vs_brute_force():
    rng = np.random.default_rng(2024)  # test_acceptance.py:47-67 (criterion 2)
    grid = [round(1.6 + 0.05 * i, 10) for i in range(17)]
    for _ in range(10_000):
        s = int(rng.integers(100, 100_000))
        c = DualConstraint(float(rng.integers(1_000, 1_000_000)), float(rng.uniform(1e4, 1e12)),
                           float(rng.choice(grid)))
        got, _ = dual_constraint_batch(s, c)
        assert got == so.brute_force_batch(s, c.m_mem, c.m_comp, c.p)


def test_tie_reports_compute_and_floor():
    assert dual_constraint_batch(10, DualConstraint(100, 1000, 2)) == (10, Binding.COMPUTE)
    assert dual_constraint_batch(10**9, DualConstraint(1e6, 1e12, 2)) == (1, Binding.FLOOR)
    assert dual_constraint_batch(10000, DualConstraint(100000, 2e9, 2)) == (10, Binding.MEMORY)
    with pytest.raises(ValueError):
        DualConstraint(0, 1, 1)
    with pytest.raises(ValueError):
        TokenBudget(0)
    with pytest.raises(ValueError):
        dual_constraint_batch(0, DualConstraint(1, 1, 1))


@settings(max_examples=200, deadline=None)
@given(s=st.integers(1, 10**6), m_mem=st.integers(1, 10**8), m_comp=st.floats(1.0, 1e14),
       p=st.floats(1.0, 3.0))
def test_batch_monotone_in_length(s, m_mem, m_comp, p):
    c = DualConstraint(float(m_mem), m_comp, p)
    assert dual_constraint_batch(s + 1, c)[0] <= dual_constraint_batch(s, c)[0]


def test_physical_load_exact():
    assert physical_load(3, 48000) == 6_912_000_000
    assert physical_load(10**6, 10**7) == 10**20


# ------------------------------------------------------------------ shapes / catalogs / plans
def test_sequence_lengths_match_reference(sampler_golden):
    for f, h, w, s in sampler_golden["sequence_length"]["lambda8"]:
        assert sequence_length(MediaShape(f, h, w), LatentGeometry()) == s
    for f, h, w, s in sampler_golden["sequence_length"]["lambda4"]:
        assert sequence_length(MediaShape(f, h, w), WAN21_GEOMETRY) == s
    # BASELINE shapes: (81, 480, 832) -> 32760 and (81, 720, 1280) -> 75600 under lambda = 4
    assert sequence_length(MediaShape(81, 480, 832), WAN21_GEOMETRY) == 32760
    assert sequence_length(MediaShape(81, 720, 1280), WAN21_GEOMETRY) == 75600


@pytest.mark.parametrize("name", ["default", "wan_l4"])
def test_catalog_and_plans_match_reference(sampler_golden, name):
    g = sampler_golden["catalogs"][name]
    cat, w, tb, dc = _catalog(name)
    assert [b.seq_len for b in cat] == g["seq_len"]
    assert [[b.shape.frames, b.shape.height, b.shape.width, b.sample_count] for b in cat] == g["shapes"]
    assert list(w) == g["weights"]
    for key, plan in (("plan_equal_token", emit_plan(cat, tb)), ("plan_dual", emit_plan(cat, dc))):
        want = g[key]
        assert [e.batch_size for e in plan.entries] == [x["batch"] for x in want]
        assert [None if e.binding is None else e.binding.value for e in plan.entries] == \
            [x["binding"] for x in want]


def test_default_plans_are_the_documented_ones():
    cat, w, tb, dc = reference_default_catalog()
    assert emit_plan(cat, tb).batch_sizes() == [300, 100, 50, 20, 10, 9]
    assert emit_plan(cat, dc).batch_sizes() == [300, 100, 32, 5, 1, 1]
    with pytest.raises(EmptyCatalog):
        emit_plan([], tb)
    with pytest.raises(EmptyCatalog):
        build_catalog([], LatentGeometry())


# ------------------------------------------------------------------ per-rank draws (bit-exact)
@pytest.mark.parametrize("name", ["default", "wan_l4"])
def test_draws_bit_exact_with_reference_run_policy(sampler_golden, name):
    g = sampler_golden["catalogs"][name]
    cat, w, tb, dc = _catalog(name)
    plans = {"equal_token": emit_plan(cat, tb), "dual": emit_plan(cat, dc)}
    for key, rec in g["draws"].items():
        policy, n, seed = key.split("/")
        nw, sd = int(n[1:]), int(seed[4:])
        # the reference's run_policy consumes N normals (jitter) after each N-rank draw
        smp = BucketSampler(cat, w, plans[policy], nw, np.random.default_rng(sd),
                            noise_draws=nw, noise_sigma=0.03)
        for step, (idx, bs, ccv) in enumerate(zip(rec["idx"], rec["batch"], rec["compute_cv"])):
            shards = smp.step()
            assert [s.bucket_index for s in shards] == idx, (key, step)
            assert [s.batch_size for s in shards] == bs
            assert compute_cv([s.load for s in shards]) == ccv


def test_sample_assignments_equals_generator_choice():
    cat, w, tb, dc = reference_default_catalog()
    plan = emit_plan(cat, dc)
    for seed in range(20):
        got = sample_assignments(cat, w, plan, 8, np.random.default_rng(seed))
        want = so.sample_indices(w, 8, np.random.default_rng(seed))
        assert [cat.index(b) for b, _ in got] == want


@pytest.mark.parametrize("name", ["default", "wan_l4"])
def test_imbalance_ab_matches_reference_run_experiment(sampler_golden, name):
    g = sampler_golden["catalogs"][name]
    cat, w, tb, dc = _catalog(name)
    for n, summary in g["experiments"].items():
        r = compare_policies(cat, w, emit_plan(cat, tb), emit_plan(cat, dc), int(n), 500, 42)
        for pol, ref_key in (("equal_token", "policy_a"), ("dual", "policy_b")):
            ref = summary[ref_key]
            assert r[pol]["mean_compute_cv"] == ref["mean_compute_cv"], (n, pol)
            assert r[pol]["mean_compute_cv_range"] == ref["mean_compute_cv_range"]
            assert r[pol]["mean_cv_step"] == pytest.approx(ref["mean_cv_step"], rel=1e-12)
            assert r[pol]["mean_t_sync"] == pytest.approx(ref["mean_t_sync"], rel=1e-12)
            assert r[pol]["tokens_per_sec"] == pytest.approx(ref["tokens_per_sec"], rel=1e-12)


def test_headline_imbalance_8_ranks():
    """at 8 ranks compute_cv 102.32 % (equal token) -> 40.77 % (dual)."""
    cat, w, tb, dc = reference_default_catalog()
    r = compare_policies(cat, w, emit_plan(cat, tb), emit_plan(cat, dc), 8, 500, 42)
    assert r["equal_token"]["mean_compute_cv"] == pytest.approx(102.32, abs=0.01)
    assert r["dual"]["mean_compute_cv"] == pytest.approx(40.77, abs=0.01)
    assert r["compute_cv_reduction"] >= 0.40  # acceptance criterion 5


# ------------------------------------------------------------------ reference behaviour ports
def test_single_bucket_zero_weight_lln_and_mismatch():
    cat, w, tb, dc = reference_default_catalog()
    plan = emit_plan(cat, tb)
    out = sample_assignments([cat[0]], [1.0], plan, 8, np.random.default_rng(0))
    assert all(a == out[0] for a in out)
    out = sample_assignments(cat[:2], [1.0, 0.0], plan, 1000, np.random.default_rng(1))
    assert all(b == cat[0] for b, _ in out)
    out = sample_assignments(cat, w, plan, 10_000, np.random.default_rng(42))
    for b, wt in zip(cat, w):
        assert abs(sum(1 for x, _ in out if x == b) / 10_000 - wt) <= 0.02
    with pytest.raises(PlanMismatch):
        sample_assignments(cat, w[:-1], plan, 4, np.random.default_rng(0))
    with pytest.raises(ValueError):
        sample_assignments(cat, [0.5] * len(cat), plan, 4, np.random.default_rng(0))
    other = emit_plan([Bucket(MediaShape(1, 16, 16), 1, 1)], tb)
    with pytest.raises(PlanMismatch):
        sample_assignments(cat, w, other, 4, np.random.default_rng(0))


def test_metrics_examples_and_errors():
    assert cv_step([100, 80]) == pytest.approx(0.2)
    assert cv_step([7, 7, 7]) == 0.0
    assert compute_cv([5, 5]) == 0.0
    with pytest.raises(AllZero):
        cv_step([0, 0])
    with pytest.raises(ZeroMean):
        compute_cv([0, 0])
