"""Central finite-difference verification of the GPU backward (reference: adaln/__init__.py:178-296).

Same contract as the reference's ``gradcheck``: for every (N, D) it draws x, scale=0.1*N(0,1),
shift=0.1*N(0,1), dy from ``np.random.default_rng(seed)`` in the reference's order, runs both
backward variants (naive and d-tile), and compares dx/dscale/dshift against central differences
of <dy, y> with the reference's tolerance convention ``max|a-r| / max|r|`` (:217-219).
Per-coordinate differences when N*D <= 8192, otherwise 16 random directional probes for dx
(:182-185, :236-253).

Everything runs in fp64 on the GPU.  The perturbed forward evaluations are batched through the
kernel's per-sample modulation layout ([B, S, D] x with [B, D] scale/shift) instead of one
launch per coordinate.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

DEFAULT_SIZES = ((8, 16), (64, 128), (512, 256), (4096, 64))

_COORD_LIMIT = 8192
_NUM_PROBES = 16
_BATCH_BYTES = 128 << 20


@dataclass(frozen=True)
class GradcheckReport:
    entries: tuple
    tolerance: float

    @property
    def passed(self) -> bool:
        return all(e["pass"] for e in self.entries)


def _max_rel_err(analytic, reference) -> float:
    a = np.asarray(analytic, dtype=np.float64)
    r = np.asarray(reference, dtype=np.float64)
    denom = max(float(np.abs(r).max()), 1e-12)
    return float(np.abs(a - r).max()) / denom


def _fd_dx_coordinates(x, scale, shift, dy, eps, h):
    """d<dy,y>/dx[i,j] by central differences; rows are independent, so only row i's term moves."""
    from ._ops import fused_forward

    n, d = x.shape
    eye = torch.eye(d, dtype=x.dtype, device=x.device) * h
    out = torch.empty((n, d), dtype=x.dtype, device=x.device)
    rows_per = max(1, _BATCH_BYTES // (2 * d * d * 8))
    for i0 in range(0, n, rows_per):
        xs = x[i0:i0 + rows_per]
        k = xs.shape[0]
        pert = torch.cat([xs[:, None, :] + eye, xs[:, None, :] - eye], 0).reshape(-1, d)
        y = fused_forward(pert.contiguous(), scale, shift, eps)[0].reshape(2, k, d, d)
        w = dy[i0:i0 + k, None, :]
        out[i0:i0 + k] = ((y[0] * w).sum(-1) - (y[1] * w).sum(-1)) / (2.0 * h)
    return out


def _fd_modulation(x, scale, shift, dy, eps, h, which: str):
    """d<dy,y>/d(scale|shift)[j], all j batched as per-sample modulation vectors."""
    from ._ops import fused_forward

    n, d = x.shape
    out = torch.empty(d, dtype=x.dtype, device=x.device)
    per = max(1, _BATCH_BYTES // (2 * n * d * 8))
    eye = torch.eye(d, dtype=x.dtype, device=x.device) * h
    for j0 in range(0, d, per):
        e = eye[j0:j0 + per]
        k = e.shape[0]
        xb = x.expand(2 * k, n, d).contiguous()
        sc = scale.expand(2 * k, d).clone()
        sh = shift.expand(2 * k, d).clone()
        tgt = sc if which == "scale" else sh
        tgt[:k] += e
        tgt[k:] -= e
        y = fused_forward(xb, sc, sh, eps)[0]
        loss = (y * dy).sum(dim=(1, 2))
        out[j0:j0 + k] = (loss[:k] - loss[k:]) / (2.0 * h)
    return out


def _loss(x, scale, shift, dy, eps) -> float:
    from ._ops import fused_forward

    return float((dy * fused_forward(x, scale, shift, eps)[0]).sum())


def _check_size(n, d, tolerance, tiles, rng, eps, h, device):
    from . import TileConfig, adaln_backward_dtile, adaln_backward_naive, adaln_forward

    xn = rng.standard_normal((n, d))
    scn = 0.1 * rng.standard_normal(d)
    shn = 0.1 * rng.standard_normal(d)
    dyn = rng.standard_normal((n, d))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
    x, scale, shift, dy = t(xn), t(scn), t(shn), t(dyn)
    out = adaln_forward(x, scale, shift, eps)
    variants = {
        "naive": adaln_backward_naive(dy, x, scale, out.mu, out.rstd),
        "dtile": adaln_backward_dtile(dy, x, scale, out.mu, out.rstd, tiles),
    }
    if n * d <= _COORD_LIMIT:
        fd_dx = _fd_dx_coordinates(x, scale, shift, dy, eps, h).cpu().numpy()
        dx_err = {k: _max_rel_err(g.dx.cpu().numpy(), fd_dx) for k, g in variants.items()}
    else:
        dx_err = {k: 0.0 for k in variants}
        for _ in range(_NUM_PROBES):
            v = rng.standard_normal((n, d))
            v /= np.linalg.norm(v)
            vt = t(v)
            fd = (_loss(x + h * vt, scale, shift, dy, eps)
                  - _loss(x - h * vt, scale, shift, dy, eps)) / (2.0 * h)
            denom = max(abs(fd), 1e-12)
            for k, g in variants.items():
                err = abs(float((g.dx * vt).sum()) - fd) / denom
                dx_err[k] = max(dx_err[k], err)
    fd_dscale = _fd_modulation(x, scale, shift, dy, eps, h, "scale").cpu().numpy()
    fd_dshift = _fd_modulation(x, scale, shift, dy, eps, h, "shift").cpu().numpy()
    entries = []
    for name, g in variants.items():
        for tensor, err in (
            ("dx", dx_err[name]),
            ("dscale", _max_rel_err(g.dscale.cpu().numpy(), fd_dscale)),
            ("dshift", _max_rel_err(g.dshift.cpu().numpy(), fd_dshift)),
        ):
            entries.append({"n": n, "d": d, "variant": name, "tensor": tensor,
                            "max_rel_err": err, "pass": err <= tolerance})
    return entries


def gradcheck(sizes=DEFAULT_SIZES, tolerance: float = 1e-4, tiles=None, fp32_accum: bool = False,
              eps: float = 1e-6, step: float = 1e-3, seed: int = 0) -> GradcheckReport:
    """Central finite-difference verification of both backward variants (reference :278-296)."""
    from . import TileConfig

    del fp32_accum  # accumulation precision is fixed on the GPU (see adaln_backward_dtile)
    if not sizes:
        raise ValueError("sizes must be non-empty")
    device = torch.device("cuda", torch.cuda.current_device())
    rng = np.random.default_rng(seed)
    entries = []
    for n, d in sizes:
        cfg = tiles or TileConfig(d_tile=min(32, d), n_tile=min(128, n))
        cfg = TileConfig(min(cfg.d_tile, d), min(cfg.n_tile, n))
        entries.extend(_check_size(n, d, tolerance, cfg, rng, eps, step, device))
    return GradcheckReport(entries=tuple(entries), tolerance=tolerance)
