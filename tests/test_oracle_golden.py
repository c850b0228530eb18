"""Pin the CPU oracle against the reference's own outputs (tests/golden/, made by the reference).

The oracle restates _kernels_numba.py in C; with the same association order and no FMA
contraction it must agree with the numba reference BIT FOR BIT.
"""

import numpy as np
import pytest

import oracle
from oracle import sampler_oracle as so


def _cases(g):
    return [str(c) for c in g["__cases__"]]


def test_golden_has_cases(adaln_golden):
    assert len(_cases(adaln_golden)) >= 15


@pytest.mark.parametrize("threads", [1, 3])
def test_oracle_forward_bitexact(adaln_golden, threads):
    g = adaln_golden
    for c in _cases(g):
        p = c + "/"
        y, mu, rstd = oracle.forward(g[p + "x"], g[p + "scale"], g[p + "shift"],
                                     float(g[p + "eps"]), threads)
        assert np.array_equal(y, g[p + "y"]), c
        assert np.array_equal(mu, g[p + "mu"]), c
        assert np.array_equal(rstd, g[p + "rstd"]), c


@pytest.mark.parametrize("threads", [1, 4])
def test_oracle_backward_naive_bitexact(adaln_golden, threads):
    g = adaln_golden
    for c in _cases(g):
        p = c + "/"
        dx, dsc, dsh = oracle.backward_naive(g[p + "dy"], g[p + "x"], g[p + "scale"],
                                             g[p + "mu"], g[p + "rstd"], threads)
        assert np.array_equal(dx, g[p + "dx"]), c
        assert np.array_equal(dsc, g[p + "dscale"]), c
        assert np.array_equal(dsh, g[p + "dshift"]), c


def test_oracle_dtile_bitexact(adaln_golden):
    g = adaln_golden
    for c in _cases(g):
        p = c + "/"
        for dt, nt in g[p + "tiles"]:
            for acc in (0, 1):
                dsc, dsh = oracle.dtile_reduce(g[p + "dy"], g[p + "x"], g[p + "mu"], g[p + "rstd"],
                                               int(dt), int(nt), bool(acc), threads=2)
                q = f"{p}dtile_{dt}_{nt}_{acc}/"
                assert np.array_equal(dsc, g[q + "dscale"]), (c, dt, nt, acc)
                assert np.array_equal(dsh, g[q + "dshift"]), (c, dt, nt, acc)


def test_oracle_hand_example(adaln_golden):
    # test_adaln.py:57-64: mu = [1.5, 4.0]
    y, mu, rstd = oracle.forward([[1.0, 2.0], [3.0, 5.0]], [0.5, -0.5], [1.0, 2.0], 1e-6)
    assert mu.tolist() == [1.5, 4.0]
    assert (rstd > 0).all()
    np.testing.assert_allclose(y, [[-0.49999700000900016, 2.499999000003],
                                   [-0.49999925000056233, 2.4999997500001876]], rtol=1e-15)


def test_oracle_as_f64_flags_nonfinite():
    a = np.array([1.0, np.nan, 2.0], dtype=np.float32)
    out, bad = oracle.as_f64(a, threads=2)
    assert bad and out[0] == 1.0
    bf = np.array([0x3F80, 0x7F80], dtype=np.uint16)  # 1.0, +inf in bf16
    out, bad = oracle.as_f64(bf)
    assert bad and out[0] == 1.0 and np.isinf(out[1])
    out, bad = oracle.as_f64(np.ones(1000, dtype=np.float32), threads=4)
    assert not bad and out.sum() == 1000.0


# ------------------------------------------------------------------ sampler oracle
def test_sampler_oracle_batch_rule(sampler_golden):
    for s, m_mem, m_comp, p, b, binding in sampler_golden["dual_constraint_batch"]:
        assert so.dual_constraint_batch(s, m_mem, m_comp, p) == (b, binding)
    for s, m_mem, m_comp, p, b, _ in sampler_golden["dual_constraint_batch"][:2000]:
        assert so.brute_force_batch(s, m_mem, m_comp, p) == b
    for s, t, b in sampler_golden["equal_token_batch"]:
        assert so.equal_token_batch(s, t) == b


def test_sampler_oracle_draws(sampler_golden):
    for cname, cat in sampler_golden["catalogs"].items():
        for key, rec in cat["draws"].items():
            policy, n, seed = key.split("/")
            nw, sd = int(n[1:]), int(seed[4:])
            idx = so.run_policy_indices(cat["weights"], nw, len(rec["idx"]),
                                        np.random.default_rng(sd))
            assert idx == rec["idx"], (cname, key)
            seqs = cat["seq_len"]
            plan = [e["batch"] for e in cat[f"plan_{policy}"]]
            for step, row in enumerate(idx):
                loads = [plan[i] * seqs[i] ** 2 for i in row]
                assert so.compute_cv(loads) == rec["compute_cv"][step]
