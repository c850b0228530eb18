"""Round-2 parity additions (VERDICT r1 "fill the parity holes"):

* adversarial 16-bit rows for the statistics (first-element outlier, large offsets, near-constant
  rows) on every forward flavour that takes them (rows16 at D=5120, rows2 at D=1536, the ring
  kernel at D=8192);
* every cfg3 length S in {14040, 20280, 46800, 61200, 75600} at D=5120: all row statistics, the
  full dscale/dshift, sampled rows of y / dx against the oracle;
* the reference's single-tile property (pkg/tests/test_adaln.py:128-135): a d-tile backward with
  one tile is bit-identical to the naive backward in fp64;
* the deterministic backward (the reference-facing API's) at full cfg2, and bitwise run to run.

Oracle: oracle/ (the C restatement of _kernels_numba.py, pinned to the reference's outputs by
tests/test_oracle_golden.py) on the exact rounded 16-bit inputs, upcast to f64.
"""

import numpy as np
import pytest
import torch

import oracle
from conftest import max_rel_err
from paper_2605_17923_b200.adaln import (TileConfig, adaln_backward_dtile, adaln_backward_naive,
                                         adaln_forward)
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward

pytestmark = pytest.mark.gpu


def f64(t):
    return t.detach().double().cpu().numpy()


def _adversarial(kind, b, s, d, dtype, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randn(b, s, d, generator=g)
    if kind == "first_outlier":
        x[:, :, 0] = 1000.0
    elif kind == "offset50":
        x = x + 50.0
    elif kind == "offset1000":
        x = x + 1000.0
    elif kind == "near_constant":
        x = 3.0 + 1e-3 * x
    elif kind == "outlier_mid":
        x[:, :, d // 2] = -3000.0
    return x.to(dtype)


KINDS = ["first_outlier", "offset50", "offset1000", "near_constant", "outlier_mid"]


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("d", [5120, 1536, 8192])
@pytest.mark.parametrize("kind", KINDS)
def test_adversarial_16bit_statistics(kind, d, dtype, cuda):
    if dtype == torch.float16 and kind == "offset1000" and d == 8192:
        pytest.skip("fp16 squares of 1000-offset rows are covered at D=5120/1536")
    x = _adversarial(kind, 2, 64, d, dtype, seed=d)
    g = torch.Generator(device="cpu").manual_seed(1)
    sc = (0.1 * torch.randn(2, d, generator=g)).to(dtype)
    sh = (0.1 * torch.randn(2, d, generator=g)).to(dtype)
    xd, scd, shd = x.to(cuda), sc.to(cuda), sh.to(cuda)
    y, mu, rs = fused_forward(xd, scd, shd)
    yo, muo, rso = oracle.forward_batched(f64(x), f64(sc), f64(sh), 1e-6, threads=0)
    # statistics in fp32: the mean to fp32 rounding of the row's largest element (an fp32 sum of
    # D values cannot do better: a +-1000 outlier alone carries 6e-5 of ulp), rstd to 1e-5
    # relative -- the part a one-pass E[x^2] - E[x]^2 loses on outlier rows
    xmax = np.abs(f64(x)).max(axis=-1)
    assert (np.abs(f64(mu) - muo) <= 1e-6 * np.maximum(1.0, xmax)).all(), kind
    assert max_rel_err(f64(rs), rso) <= 1e-5, kind
    assert max_rel_err(f64(y), yo) <= 2e-2, kind
    # what exact two-pass statistics achieve: the output's own 16-bit rounding
    assert max_rel_err(f64(y), yo) <= 8e-3, kind


CFG3_LONG = [14040, 20280, 46800, 61200, 75600]


@pytest.mark.slow
@pytest.mark.parametrize("S", CFG3_LONG)
def test_cfg3_long_lengths_vs_oracle(S, cuda):
    d = 5120
    g = torch.Generator(device="cpu").manual_seed(S)
    x = torch.randn(1, S, d, generator=g).to(torch.bfloat16)
    dy = torch.randn(1, S, d, generator=g).to(torch.bfloat16)
    sc = (0.1 * torch.randn(1, d, generator=g)).to(torch.bfloat16)
    sh = (0.1 * torch.randn(1, d, generator=g)).to(torch.bfloat16)
    y, mu, rs = fused_forward(x.to(cuda), sc.to(cuda), sh.to(cuda))
    dx, dsc, dsh = fused_backward(dy.to(cuda), x.to(cuda), sc.to(cuda), mu, rs)
    xn, dyn, scn, shn = f64(x)[0], f64(dy)[0], f64(sc)[0], f64(sh)[0]
    yo, muo, rso = oracle.forward(xn, scn, shn, 1e-6, threads=0)
    assert np.abs(f64(mu)[0] - muo).max() < 1e-6
    assert max_rel_err(f64(rs)[0], rso) <= 1e-5
    rows = np.random.default_rng(S).choice(S, 256, replace=False)
    assert max_rel_err(f64(y)[0][rows], yo[rows]) <= 2e-2
    dxo = oracle.backward_dx(dyn[rows], xn[rows], scn, muo[rows], rso[rows], threads=0)
    assert max_rel_err(f64(dx)[0][rows], dxo) <= 2e-2
    dsco, dsho = oracle.reduce_naive(dyn, xn, muo, rso, threads=0)
    assert max_rel_err(f64(dsc)[0], dsco) <= 1e-5
    assert max_rel_err(f64(dsh)[0], dsho) <= 1e-5


def test_single_tile_dtile_bitwise_equals_naive_f64(cuda):
    """pkg/tests/test_adaln.py:128-135 on the GPU path, fp64."""
    rng = np.random.default_rng(2)
    x = rng.standard_normal((64, 16))
    scale = 0.1 * rng.standard_normal(16)
    shift = 0.1 * rng.standard_normal(16)
    dy = rng.standard_normal((64, 16))
    out = adaln_forward(x, scale, shift)
    naive = adaln_backward_naive(dy, x, scale, out.mu, out.rstd)
    tiled = adaln_backward_dtile(dy, x, scale, out.mu, out.rstd, TileConfig(16, 64))
    assert np.array_equal(tiled.dshift, naive.dshift)
    assert np.array_equal(tiled.dscale, naive.dscale)
    np.testing.assert_array_equal(tiled.dx, naive.dx)


@pytest.mark.slow
def test_deterministic_backward_full_cfg2(cuda):
    """The partition the reference-facing API runs, at the Wan-14B shape: full dscale/dshift and
    sampled dx against the oracle, and bit-identical outputs over repeated calls."""
    g = torch.Generator(device="cpu").manual_seed(11)
    x = torch.randn(1, 32760, 5120, generator=g).to(torch.bfloat16)
    dy = torch.randn(1, 32760, 5120, generator=g).to(torch.bfloat16)
    sc = (0.1 * torch.randn(1, 5120, generator=g)).to(torch.bfloat16)
    sh = (0.1 * torch.randn(1, 5120, generator=g)).to(torch.bfloat16)
    xd, dyd, scd, shd = (t.to(cuda) for t in (x, dy, sc, sh))
    y, mu, rs = fused_forward(xd, scd, shd)
    first = fused_backward(dyd, xd, scd, mu, rs, deterministic=True)
    for _ in range(3):
        again = fused_backward(dyd, xd, scd, mu, rs, deterministic=True)
        for a, b in zip(first, again):
            assert torch.equal(a, b)
    dx, dsc, dsh = first
    xn, dyn, scn = f64(x)[0], f64(dy)[0], f64(sc)[0]
    muo, rso = f64(mu)[0], f64(rs)[0]
    dsco, dsho = oracle.reduce_naive(dyn, xn, muo, rso, threads=0)
    assert max_rel_err(f64(dsc)[0], dsco) <= 1e-5
    assert max_rel_err(f64(dsh)[0], dsho) <= 1e-5
    rows = np.random.default_rng(0).choice(32760, 256, replace=False)
    dxo = oracle.backward_dx(dyn[rows], xn[rows], scn, muo[rows], rso[rows], threads=0)
    assert max_rel_err(f64(dx)[0][rows], dxo) <= 2e-2


def test_dynamic_backward_dx_identical_to_deterministic(cuda):
    """The dynamic tail changes only the summation order of the last group's dscale/dshift; dx is
    bit-identical to the static partition's."""
    g = torch.Generator(device="cpu").manual_seed(12)
    x = torch.randn(1, 20000, 5120, generator=g).to(torch.bfloat16).to(cuda)
    dy = torch.randn(1, 20000, 5120, generator=g).to(torch.bfloat16).to(cuda)
    sc = (0.1 * torch.randn(1, 5120, generator=g)).to(torch.bfloat16).to(cuda)
    y, mu, rs = fused_forward(x, sc, sc)
    a = fused_backward(dy, x, sc, mu, rs, deterministic=True)
    b = fused_backward(dy, x, sc, mu, rs, deterministic=False)
    assert torch.equal(a[0], b[0])
    # fp32 partial sums in another order: agreement to fp32 accumulation level (max-norm)
    assert max_rel_err(f64(b[1]), f64(a[1])) <= 2e-6
    assert max_rel_err(f64(b[2]), f64(a[2])) <= 2e-6
