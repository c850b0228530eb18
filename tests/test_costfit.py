"""Cost-model fitting (costfit.py) vs the reference's outputs on the same trials."""

import pytest

from paper_2605_17923_b200.catalogs import reference_default_catalog
from paper_2605_17923_b200.costfit import (
    CostModel, DegenerateFit, GridSpec, InsufficientData, TargetBelowOverhead, Trial, ZeroSlope,
    calibrated_dual_constraint, correlation_report, derive_m_comp, fit_cost_model,
    generate_sweep, r_squared)
from paper_2605_17923_b200.scheduler import emit_plan


def _trials(rows):
    return [Trial(int(b), int(s), float(t)) for b, s, t in rows]


def test_recovery_matches_reference(sampler_golden):
    for case in sampler_golden["costfit"]["recovery"]:
        m = fit_cost_model(_trials(case["trials"]))
        assert m.p == case["fit"][2]
        assert m.a == pytest.approx(case["fit"][0], rel=1e-12, abs=1e-12)
        assert m.b == pytest.approx(case["fit"][1], rel=1e-12)
        assert m.r2 == pytest.approx(case["fit"][3], abs=1e-12)
        assert derive_m_comp(m, 62.0) == pytest.approx(case["m_comp_62"], rel=1e-12)


def test_noisy_fit_and_correlations_match_reference(sampler_golden):
    g = sampler_golden["costfit"]
    trials = _trials(g["noisy"]["trials"])
    m = fit_cost_model(trials)
    assert [m.p] == [g["noisy"]["fit"][2]]
    assert m.r2 == pytest.approx(g["noisy"]["fit"][3], abs=1e-12)
    c = correlation_report(trials, 2.0)
    assert c["corr_load"] == pytest.approx(g["noisy"]["corr"]["corr_load"], abs=1e-12)
    assert c["corr_tokens"] == pytest.approx(g["noisy"]["corr"]["corr_tokens"], abs=1e-12)
    wide = GridSpec(1.0, 2.4, 0.05)
    assert wide.values() == g["grids"]["wide"]["values"]
    assert fit_cost_model(trials, wide).p == g["grids"]["wide"]["fit"][2]


def test_generate_sweep_matches_reference(sampler_golden):
    cat, _, _, _ = reference_default_catalog()
    assert [list(r) for r in generate_sweep(cat).trials] == sampler_golden["costfit"]["sweep_default"]


def test_errors():
    with pytest.raises(InsufficientData):
        fit_cost_model([Trial(1, 10, 1.0)] * 2)
    with pytest.raises(DegenerateFit):
        fit_cost_model([Trial(1, 10, 1.0), Trial(2, 10, 1.0), Trial(3, 10, 1.0)])
    with pytest.raises(ZeroSlope):
        derive_m_comp(CostModel(1.0, 0.0, 2.0, 1.0), 5.0)
    with pytest.raises(TargetBelowOverhead):
        derive_m_comp(CostModel(10.0, 1.0, 2.0, 1.0), 5.0)
    with pytest.raises(ValueError):
        Trial(1, 1, 0.0)
    assert r_squared([1, 2, 3], [1, 2, 3]) == 1.0


def test_calibrated_plan_equalises_predicted_time():
    cat, w, tb, dc = reference_default_catalog()
    model = CostModel(a=0.005, b=2e-9, p=1.4, r2=0.99)
    plan = emit_plan(cat, calibrated_dual_constraint(model, cat, 480_000))
    times = [model.predict(e.batch_size, e.bucket.seq_len) for e in plan.entries]
    target = model.predict(1, max(b.seq_len for b in cat))
    assert all(t <= target * (1 + 1e-6) for t in times)
    # the longest bucket runs B = 1; every compute-bound bucket is within one sample of target
    assert plan.entries[-1].batch_size == 1
    for e, t in zip(plan.entries, times):
        if e.binding.value == "compute":
            assert model.predict(e.batch_size + 1, e.bucket.seq_len) > target


def test_quadratic_model_fits_measured_b200_block_trials():
    """Trials measured on a B200 (profiles/r1_dit_calibration.json) -- linear + quadratic."""
    from paper_2605_17923_b200.costfit import fit_quadratic_cost_model, time_balanced_plan

    rows = [[1, 1600, 0.002236], [2, 1600, 0.002954], [1, 4800, 0.003182], [2, 4800, 0.005478],
            [1, 9600, 0.006096], [2, 9600, 0.010995], [1, 24000, 0.018733], [2, 24000, 0.03823],
            [3, 24000, 0.056679], [4, 24000, 0.074578], [1, 48000, 0.058422],
            [2, 48000, 0.115555], [3, 48000, 0.17569], [4, 48000, 0.235084],
            [1, 52800, 0.069602], [2, 52800, 0.137786], [3, 52800, 0.210791],
            [4, 52800, 0.280007], [300, 1600, 0.19181], [100, 4800, 0.219466],
            [50, 9600, 0.259281], [20, 24000, 0.386167], [10, 48000, 0.59469],
            [9, 52800, 0.638658]]
    trials = _trials(rows)
    q = fit_quadratic_cost_model(trials)
    pw = fit_cost_model(trials, GridSpec(1.0, 2.4, 0.05))
    assert q.r2 > 0.999 and q.r2 > pw.r2 and q.c1 > 0 and q.c2 > 0
    cat, _, _, _ = reference_default_catalog()
    plan = time_balanced_plan(q, cat, 480_000)
    pred = [q.predict(e.batch_size, e.bucket.seq_len) for e in plan.entries]
    target = q.predict(1, 52800)
    assert max(pred) <= target * (1 + 1e-6)
    assert plan.batch_sizes() == [110, 32, 13, 3, 1, 1]
