"""Generate the golden fixtures by running the REFERENCE implementation (this container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Imports the reference package in place from /root/reference/pkg/src (read-only; numba backend,
as shipped) and records its outputs on fixed inputs:

* adaln_golden.npz   -- adaln_forward / adaln_backward_naive / adaln_backward_dtile (f64 and
                        fp32-accumulator variants) on the reference test suite's cases
                        (test_adaln.py rand_case seeds, hand example, degenerate cases) plus a
                        Wan-width (D=5120) bf16-rounded case and a +50-offset case.
* sampler_golden.json -- dual_constraint_batch / equal_token_batch / emit_plan results,
                        sample_assignments draws as consumed by run_policy (choice + normal per
                        step), per-step compute_cv, and run_experiment summaries at 2/4/8/16 ranks.

The fixtures are committed; /root/reference does not exist on the GPU box.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF_SRC)

from adaptiveload import adaln  # noqa: E402
from adaptiveload.cluster_sim import (  # noqa: E402
    ClusterConfig, compute_cv, default_catalog, default_dual_constraint, default_token_budget,
    run_experiment, run_policy)
from adaptiveload.scheduler import (  # noqa: E402
    DualConstraint, TokenBudget, dual_constraint_batch, emit_plan, equal_token_batch)
from adaptiveload.shapes import LatentGeometry, MediaShape, build_catalog, sequence_length  # noqa: E402

assert adaln.BACKEND == "numba", adaln.BACKEND


def rand_case(n, d, seed=0):  # test_adaln.py:20-27
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((n, d)), 0.5 * rng.standard_normal(d),
            0.5 * rng.standard_normal(d), rng.standard_normal((n, d)))


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float64 (what the GPU sees, upcast)."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def adaln_cases():
    cases = {}
    x = np.array([[1.0, 2.0], [3.0, 5.0]])
    cases["hand"] = (x, np.array([0.5, -0.5]), np.array([1.0, 2.0]),
                     np.array([[0.3, -1.2], [0.7, 2.0]]), 1e-6)
    for (n, d, seed) in [(5, 8, 0), (64, 16, 2), (32, 8, 4), (64, 32, 3), (128, 32, 8),
                         (7, 4, 0), (1, 16, 0), (8, 16, 1), (4, 6, 0), (512, 64, 5)]:
        xx, sc, sh, dy = rand_case(n, d, seed)
        cases[f"rand_{n}x{d}_s{seed}"] = (xx, sc, sh, dy, 1e-6)
    cases["d1"] = (np.array([[3.0], [5.0], [-1.0]]), np.array([0.7]), np.array([2.0]),
                   np.ones((3, 1)), 1e-6)
    rng = np.random.default_rng(10)
    x6 = rng.standard_normal((6, 5))
    cases["scale_minus1"] = (x6, -np.ones(5), np.zeros(5), rng.standard_normal((6, 5)), 1e-6)
    rng = np.random.default_rng(2605)
    cases["wan_bf16_3x5120"] = (bf16_round(rng.standard_normal((3, 5120))),
                                bf16_round(0.1 * rng.standard_normal(5120)),
                                bf16_round(0.1 * rng.standard_normal(5120)),
                                bf16_round(rng.standard_normal((3, 5120))), 1e-6)
    rng = np.random.default_rng(50)
    cases["offset50_96x320"] = (50.0 + rng.standard_normal((96, 320)),
                                0.3 * rng.standard_normal(320), 0.3 * rng.standard_normal(320),
                                rng.standard_normal((96, 320)), 1e-6)
    return cases


TILES = [(1, 1), (3, 7), (8, 128), (64, 1), (64, 4096), (13, 999)]


def make_adaln():
    arrays = {}
    names = []
    for name, (x, sc, sh, dy, eps) in adaln_cases().items():
        n, d = x.shape
        out = adaln.adaln_forward(x, sc, sh, eps)
        g = adaln.adaln_backward_naive(dy, x, sc, out.mu, out.rstd)
        p = f"{name}/"
        arrays.update({p + "x": x, p + "scale": sc, p + "shift": sh, p + "dy": dy,
                       p + "eps": np.array(eps), p + "y": out.y, p + "mu": out.mu,
                       p + "rstd": out.rstd, p + "dx": g.dx, p + "dscale": g.dscale,
                       p + "dshift": g.dshift})
        tiles = sorted({(min(a, d), min(b, n)) for a, b in TILES})
        arrays[p + "tiles"] = np.array(tiles, dtype=np.int64)
        for (dt, nt) in tiles:
            for acc in (0, 1):
                gt = adaln.adaln_backward_dtile(dy, x, sc, out.mu, out.rstd,
                                                adaln.TileConfig(dt, nt), fp32_accum=bool(acc))
                q = f"{p}dtile_{dt}_{nt}_{acc}/"
                arrays[q + "dscale"] = gt.dscale
                arrays[q + "dshift"] = gt.dshift
                if acc == 0 and (dt, nt) == tiles[0]:
                    arrays[p + "dtile_dx"] = gt.dx
        names.append(name)
    arrays["__cases__"] = np.array(names)
    np.savez_compressed(OUT / "adaln_golden.npz", **arrays)


def wan_catalog_shapes():
    """Wan-2.1 lambda=4 shapes: 480x832 and 720x1280 stills and 17..81-frame videos."""
    shapes = [(MediaShape(1, 480, 832), 40), (MediaShape(1, 720, 1280), 20)]
    for f, c in [(17, 24), (33, 16), (49, 10), (65, 6), (81, 4)]:
        shapes.append((MediaShape(f, 480, 832), c))
    for f, c in [(17, 8), (33, 5), (49, 3), (81, 2)]:
        shapes.append((MediaShape(f, 720, 1280), c))
    return shapes


def plan_json(plan):
    return [{"seq_len": e.bucket.seq_len, "batch": e.batch_size,
             "binding": None if e.binding is None else e.binding.value} for e in plan.entries]


def make_sampler():
    out = {}
    rng = np.random.default_rng(11)
    grid = [round(1.6 + 0.05 * i, 10) for i in range(17)]
    cases = []
    for _ in range(2000):
        s = int(rng.integers(100, 100_000))
        c = (float(rng.integers(1_000, 1_000_000)), float(rng.uniform(1e4, 1e12)),
             float(rng.choice(grid)))
        b, binding = dual_constraint_batch(s, DualConstraint(*c))
        cases.append([s, *c, b, binding.value])
    for s, c in [(10000, (100000, 2e9, 2)), (10**9, (1e6, 1e12, 2)), (48000, (1e6, 1.2e10, 2)),
                 (10, (100, 1000, 2)), (1, (48000, 48000, 1.0)), (52801, (48000, 48000, 1.0))]:
        b, binding = dual_constraint_batch(s, DualConstraint(*map(float, c)))
        cases.append([s, *map(float, c), b, binding.value])
    out["dual_constraint_batch"] = cases
    out["equal_token_batch"] = [[s, t, equal_token_batch(s, TokenBudget(t))]
                                for s, t in [(1600, 48000), (48000, 48000), (100000, 48000),
                                             (1, 7), (7, 7), (480000, 480000), (1560, 480000)]]

    catalogs = {}
    cat, w = default_catalog()
    catalogs["default"] = (cat, w, LatentGeometry(), default_token_budget(),
                           default_dual_constraint())
    geom4 = LatentGeometry(temporal_factor=4)
    wcat = build_catalog(wan_catalog_shapes(), geom4)
    tot = sum(b.sample_count for b in wcat)
    catalogs["wan_l4"] = (wcat, [b.sample_count / tot for b in wcat], geom4,
                          TokenBudget(480_000), DualConstraint(480_000, 3e9, 2.0))
    out["catalogs"] = {}
    for cname, (cat, w, geom, tb, dc) in catalogs.items():
        plan_a = emit_plan(cat, tb)
        plan_b = emit_plan(cat, dc)
        entry = {
            "geometry": [geom.temporal_factor, geom.width_factor, geom.height_factor,
                         geom.text_tokens],
            "shapes": [[b.shape.frames, b.shape.height, b.shape.width, b.sample_count]
                       for b in cat],
            "seq_len": [b.seq_len for b in cat],
            "weights": list(w),
            "token_budget": tb.budget,
            "dual": [dc.m_mem, dc.m_comp, dc.p],
            "plan_equal_token": plan_json(plan_a),
            "plan_dual": plan_json(plan_b),
            "draws": {},
        }
        index = {b.shape: i for i, b in enumerate(cat)}
        for policy, plan in (("equal_token", plan_a), ("dual", plan_b)):
            for nw in (2, 8):
                for seed in (0, 42):
                    cfg = ClusterConfig(num_workers=nw, steps=40, seed=seed)
                    series, recs, _ = run_policy(cat, w, plan, cfg, np.random.default_rng(seed),
                                                 geom, collect_records=True)
                    idx = [[index[wk.bucket.shape] for wk in r.per_worker] for r in recs]
                    bs = [[wk.batch_size for wk in r.per_worker] for r in recs]
                    entry["draws"][f"{policy}/n{nw}/seed{seed}"] = {
                        "idx": idx, "batch": bs,
                        "compute_cv": [float(v) for v in series.compute_cv],
                        "compute_cv_range": [float(v) for v in series.compute_cv_range],
                    }
        entry["experiments"] = {}
        for nw in (2, 4, 8, 16):
            res = run_experiment(cat, w, plan_a, plan_b,
                                 ClusterConfig(num_workers=nw, steps=500, seed=42), geom)
            entry["experiments"][str(nw)] = res.summary
        out["catalogs"][cname] = entry

    shapes = [(1, 640, 640), (17, 640, 640), (233, 640, 640), (257, 640, 640), (1, 480, 832),
              (81, 480, 832), (81, 720, 1280), (1, 16, 16)]
    out["sequence_length"] = {
        "lambda8": [[*s, sequence_length(MediaShape(*s), LatentGeometry())]
                    for s in shapes if (s[0] - 1) % 8 == 0],
        "lambda4": [[*s, sequence_length(MediaShape(*s), geom4)] for s in shapes],
    }
    out["costfit"] = make_costfit()
    (OUT / "sampler_golden.json").write_text(json.dumps(out, indent=1, sort_keys=True))


def make_costfit():
    from adaptiveload.costfit import (GridSpec, Trial, correlation_report, derive_m_comp,
                                      fit_cost_model, generate_sweep)

    res = {"recovery": [], "grids": {}}
    pairs = [(bb, ss) for bb in (1, 2, 3) for ss in (8000, 24000, 48000)]
    for p_true in GridSpec().values():  # test_acceptance.py:69-83 (criterion 3)
        trials = [Trial(b, s, 2.0 + 1e-9 * b * float(s) ** p_true) for b, s in pairs]
        m = fit_cost_model(trials)
        res["recovery"].append({"trials": [[t.batch, t.seq_len, t.step_time] for t in trials],
                                "fit": [m.a, m.b, m.p, m.r2],
                                "m_comp_62": derive_m_comp(m, 62.0)})
    rng = np.random.default_rng(7)
    noisy = []
    for _ in range(100):
        b = int(rng.integers(1, 5))
        s = int(rng.choice([1600, 4800, 9600, 24000, 48000, 52800]))
        noisy.append(Trial(b, s, float((2.0 + 1e-9 * b * s**2) * (1 + rng.normal(0, 0.05)))))
    m = fit_cost_model(noisy)
    res["noisy"] = {"trials": [[t.batch, t.seq_len, t.step_time] for t in noisy],
                    "fit": [m.a, m.b, m.p, m.r2], "corr": correlation_report(noisy, 2.0)}
    wide = GridSpec(1.0, 2.4, 0.05)
    m = fit_cost_model(noisy, wide)
    res["grids"]["wide"] = {"values": wide.values(), "fit": [m.a, m.b, m.p, m.r2]}
    cat, _ = default_catalog()
    res["sweep_default"] = [list(r) for r in generate_sweep(cat).trials]
    return res


def make_io():
    """Reference-written plan / model / trace / metrics files (tests/golden/io/)."""
    from adaptiveload import io as rio
    from adaptiveload.cluster_sim import run_experiment
    from adaptiveload.costfit import Trial, fit_cost_model
    from adaptiveload.manifest import RunManifest

    d = OUT / "io"
    d.mkdir(exist_ok=True)
    cat, w = default_catalog()
    man = RunManifest(command="plan", inputs=["catalog.json"], outputs=["plan.json"], seed=42,
                      config_digest="0" * 64)
    rio.save_plan(d / "plan_dual.json", emit_plan(cat, default_dual_constraint()), man)
    rio.save_plan(d / "plan_equal_token.json", emit_plan(cat, default_token_budget()), man)
    trials = [Trial(b, s, 2.0 + 1e-9 * b * s ** 2) for b, s in ((1, 1600), (3, 24000), (1, 52800))]
    rio.save_trace(d / "trace.jsonl", trials, workers=[0, 1, 0])
    rio.save_model(d / "model.json", fit_cost_model(trials), man)
    res = run_experiment(cat, w, emit_plan(cat, default_token_budget()),
                         emit_plan(cat, default_dual_constraint()),
                         ClusterConfig(num_workers=4, steps=5, seed=42))
    rio.save_metrics_csv(d / "metrics.csv", {"equal_token": res.series_a, "dual": res.series_b})


def make_io_r2():
    """Round 2: catalog / cluster-config / summary / manifest files and config digests written
    or computed by the reference's io.py and manifest.py (tests/golden/io/)."""
    from adaptiveload import io as rio
    from adaptiveload.costfit import analyze_bottleneck
    from adaptiveload.manifest import RunManifest, config_digest

    d = OUT / "io"
    d.mkdir(exist_ok=True)
    cat, _ = default_catalog()
    rio.save_catalog(d / "catalog_default.json", cat, LatentGeometry())
    geom4 = LatentGeometry(temporal_factor=4, width_factor=16, height_factor=16, text_tokens=0)
    wan = build_catalog([(MediaShape(1, 480, 832), 40), (MediaShape(81, 480, 832), 4),
                         (MediaShape(81, 720, 1280), 2)], geom4)
    rio.save_catalog(d / "catalog_wan_l4.json", wan, geom4)
    (d / "catalog_list.json").write_text(json.dumps(
        [{"frames": 17, "height": 640, "width": 640, "count": 5},
         {"frames": 1, "height": 640, "width": 640, "count": 15}]))
    loaded = {}
    for name in ("catalog_default.json", "catalog_wan_l4.json", "catalog_list.json"):
        c, w, g = rio.load_catalog(d / name)
        loaded[name] = {"seq": [b.seq_len for b in c], "count": [b.sample_count for b in c],
                        "weights": w, "geometry": [g.temporal_factor, g.width_factor,
                                                   g.height_factor, g.text_tokens]}
    (d / "cluster_partial.json").write_text(json.dumps({"num_workers": 8, "cost": {"p": 1.5}}))
    (d / "cluster_full.json").write_text(json.dumps(
        {"num_workers": 4, "cost": {"a": 1.0, "b": 2e-9, "p": 2.2}, "noise_sigma": 0.0,
         "seed": 7, "steps": 40}))
    clusters = {}
    for name, seed in (("cluster_partial.json", None), ("cluster_full.json", None),
                       ("cluster_full.json", 99)):
        c = rio.load_cluster_config(d / name, seed_override=seed)
        clusters[f"{name}:{seed}"] = [c.num_workers, c.cost.a, c.cost.b, c.cost.p, c.noise_sigma,
                                      c.seed, c.steps]
    man = RunManifest(command="simulate", inputs=["catalog.json", "cluster.json"],
                      outputs=["summary.json"], seed=42,
                      config_digest=config_digest({"policy": "dual", "m_comp": 3e9, "p": 2.0}))
    rio.save_summary(d / "summary.json", {"cv_step": 0.25, "tokens_per_sec": 1234.5,
                                          "policies": ["equal_token", "dual"]}, man)
    rio.write_manifest_sidecar(d / "trace.jsonl", man)
    payloads = [{}, {"b": 1, "a": 2}, {"m_comp": 3e9, "p": 2.0, "policy": "dual"},
                {"nested": {"z": [1, 2.5, None], "a": True}, "s": "x"}, [3, {"k": "v"}]]
    digests = [[pl, config_digest(pl)] for pl in payloads]
    # bottleneck analysis (costfit.py:209-232) on simulator-style wait records
    from types import SimpleNamespace

    from adaptiveload.costfit import CostModel

    rng = np.random.default_rng(3)
    waits = []
    for _ in range(20):
        t = rng.exponential(0.2, 8) + 1.0
        waits.append([float(v) for v in (t.max() - t)])  # the straggler waits exactly 0
    recs = [SimpleNamespace(per_worker=[SimpleNamespace(wait_sync=v) for v in row]) for row in waits]
    bn = analyze_bottleneck(recs)
    bn2 = analyze_bottleneck(recs, CostModel(a=2.0, b=1e-9, p=2.0, r2=1.0), 62.0)

    def as_json(r):
        return {"mean_wait": [float(v) for v in r.mean_wait],
                "straggler_fraction": [float(v) for v in r.straggler_fraction],
                "suggested_m_comp": r.suggested_m_comp}

    bottleneck = {"waits": waits, "result": as_json(bn), "result_model": as_json(bn2)}
    (d / "io_r2.json").write_text(json.dumps({"loaded_catalogs": loaded, "clusters": clusters,
                                              "digests": digests, "bottleneck": bottleneck},
                                             indent=1, sort_keys=True))


if __name__ == "__main__":
    if sys.argv[1:] == ["io_r2"]:
        make_io_r2()
    else:
        make_adaln()
        make_sampler()
        make_io()
        make_io_r2()
    print("wrote", sorted(p.name for p in OUT.iterdir()))
