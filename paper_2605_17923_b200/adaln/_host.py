"""Host-buffer path: the reference-style call with torch CPU tensors, pipelined over row chunks.

The reference API takes host arrays (adaln/__init__.py:99-158), so an end-to-end call moves
every input over PCIe and every result back.  Done naively (copy in, compute, copy out) the two
PCIe directions and the kernels serialise.  Here rows are processed in ~32 MB chunks: chunk i's
inputs are copied in and computed on the current stream while chunk i-1's results drain to
pinned host memory on a second stream, so host->device and device->host traffic overlap (they
use different copy engines) and the kernels hide under the copies.

Per-chunk dscale/dshift partials are summed in a fixed order in fp64 at the end, so results are
deterministic for a given chunking.

Resident input: the reference's training pattern is forward(x) then backward(dy, x, ...), so the
device copy of x that the forward uploaded is kept (one per device) and the backward uses it
instead of moving x over PCIe a second time -- the backward then copies dy in while dx drains,
instead of 2x the bytes in one direction (cfg2: 1 006 -> 671 MB host->device per step).  Validity
follows PyTorch's own rule for saved tensors (autograd's "modified by an inplace operation"
check): the same tensor object, alive, with an unchanged version counter; writes that bypass the
version counter (e.g. through a ``.numpy()`` alias) are not seen, as with autograd.  The copy is
dropped when x is garbage-collected, replaced by the next forward, or on ``release_resident()``;
``AL_HOST_RESIDENT=0`` disables it.
"""

from __future__ import annotations

import os
import threading
import weakref

import torch

from ..errors import NonFiniteInput
from ._ops import fused_backward, fused_forward, geometry, stat_dtype

# host->device bytes per pipeline chunk (AL_HOST_CHUNK_MB overrides, A/B runs)
CHUNK_BYTES = int(float(os.environ.get("AL_HOST_CHUNK_MB", "32")) * (1 << 20))

_side_streams: dict = {}


def _side(dev: torch.device) -> torch.cuda.Stream:
    s = _side_streams.get(dev.index)
    if s is None:
        s = _side_streams[dev.index] = torch.cuda.Stream(device=dev)
    return s


def _chunks(b: int, s: int, row_bytes: int):
    """(b0, b1, s0, s1) blocks: whole samples when a sample is small, else row slices of one."""
    rows = max(1, CHUNK_BYTES // max(row_bytes, 1))
    if s >= rows:
        for bi in range(b):
            for s0 in range(0, s, rows):
                yield bi, bi + 1, s0, min(s, s0 + rows)
    else:
        per = max(1, rows // max(s, 1))
        for b0 in range(0, b, per):
            yield b0, min(b, b0 + per), 0, s


class _PinnedPool:
    """Page-locked host result buffers, reused across calls.

    A fresh ``torch.empty(pin_memory=True)`` of a few hundred MB goes through cudaHostAlloc
    whenever torch's caching host allocator has no free block of that size class, which stalls
    the call for 40-120 ms (round-1 driver e2e: 22 ms typical steps, 60-140 ms outliers).  Here
    a buffer is handed out again only once nothing outside the pool references its storage (the
    caller dropped the previous results, views and numpy aliases included), so results stay
    valid for as long as the caller keeps them; at most ``MAX_PER_SIZE`` buffers are kept per
    size, beyond that a call falls back to a one-off allocation."""

    MAX_PER_SIZE = 4

    def __init__(self):
        self._bufs: dict = {}
        self._lock = threading.Lock()

    @staticmethod
    def _free(buf: torch.Tensor) -> bool:
        # references: the pool's tensor + the temporary storage wrapper of this query
        return torch._C._storage_Use_Count(buf.untyped_storage()._cdata) <= 2

    def get(self, shape, dtype) -> torch.Tensor:
        numel = 1
        for d in shape:
            numel *= int(d)
        nbytes = max(numel * torch.empty((), dtype=dtype).element_size(), 1)
        with self._lock:
            lst = self._bufs.setdefault(nbytes, [])
            buf = next((b for b in lst if self._free(b)), None)
            if buf is None:
                buf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
                if len(lst) < self.MAX_PER_SIZE:
                    lst.append(buf)
        return buf.view(dtype)[:numel].view(shape)


_pool = _PinnedPool()


class _Resident:
    """Device copy of the last host_forward input, per device (see the module docstring)."""

    def __init__(self):
        self._e: dict = {}
        self._lock = threading.Lock()
        self.enabled = os.environ.get("AL_HOST_RESIDENT", "1") != "0"

    def put(self, x: torch.Tensor, xd: torch.Tensor, dev: torch.device) -> None:
        if not self.enabled:
            return
        idx = dev.index

        def drop(ref, idx=idx):
            with self._lock:
                e = self._e.get(idx)
                if e is not None and e[0] is ref:
                    del self._e[idx]

        with self._lock:
            self._e[idx] = (weakref.ref(x, drop), x._version, tuple(x.shape), x.dtype, xd)

    def get(self, x: torch.Tensor, dev: torch.device):
        with self._lock:
            e = self._e.get(dev.index)
        if e is None:
            return None
        ref, ver, shape, dtype, xd = e
        if ref() is x and x._version == ver and tuple(x.shape) == shape and x.dtype == dtype:
            return xd
        return None

    def clear(self) -> None:
        with self._lock:
            self._e.clear()


_resident = _Resident()


def release_resident() -> None:
    """Free the device copies the host forward keeps for a following backward."""
    _resident.clear()


def _pinned_like(shape, dtype):
    return _pool.get(tuple(shape), dtype)


def host_forward(x: torch.Tensor, scale: torch.Tensor, shift: torch.Tensor, eps: float,
                 check_finite: bool, dev: torch.device):
    g = geometry(x, scale, shift)
    B, S, D = g.batch, g.seq, g.dim
    x3 = x.contiguous().view(B, S, D)
    sdt = stat_dtype(x.dtype)
    y = _pinned_like(x.shape, x.dtype)
    mu = _pinned_like(g.stats_shape, sdt)
    rs = _pinned_like(g.stats_shape, sdt)
    y3, mu2, rs2 = y.view(B, S, D), mu.view(B, S), rs.view(B, S)
    per_sample = g.mod_stride != 0
    sc = scale.to(dev, non_blocking=True).to(x.dtype)
    sh = shift.to(dev, non_blocking=True).to(x.dtype)
    flag = torch.zeros(1, dtype=torch.int32, device=dev) if check_finite else None
    main, side = torch.cuda.current_stream(dev), _side(dev)
    # one device buffer for the whole input (chunks are views of it), kept for the backward
    xdev = torch.empty((B, S, D), dtype=x.dtype, device=dev)
    for b0, b1, s0, s1 in _chunks(B, S, D * x.element_size()):
        xd = xdev[b0:b1, s0:s1]
        xd.copy_(x3[b0:b1, s0:s1], non_blocking=True)
        scb = sc[b0:b1] if per_sample else sc
        shb = sh[b0:b1] if per_sample else sh
        yd, mud, rsd = fused_forward(xd, scb, shb, eps, flag=flag)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            y3[b0:b1, s0:s1].copy_(yd, non_blocking=True)
            mu2[b0:b1, s0:s1].copy_(mud, non_blocking=True)
            rs2[b0:b1, s0:s1].copy_(rsd, non_blocking=True)
        for t in (yd, mud, rsd):
            t.record_stream(side)
    side.synchronize()
    if flag is not None and int(flag.item()):
        raise NonFiniteInput("x/scale/shift contains NaN or Inf")
    _resident.put(x, xdev, dev)
    return y, mu, rs


def host_backward(dy: torch.Tensor, x: torch.Tensor, scale: torch.Tensor, mu: torch.Tensor,
                  rstd: torch.Tensor, d_tile: int, n_tile: int, check_finite: bool,
                  dev: torch.device):
    g = geometry(x, scale)
    B, S, D = g.batch, g.seq, g.dim
    x3, dy3 = x.contiguous().view(B, S, D), dy.contiguous().view(B, S, D)
    sdt = stat_dtype(x.dtype)
    mu2 = mu.to(sdt).contiguous().view(B, S)
    rs2 = rstd.to(sdt).contiguous().view(B, S)
    dx = _pinned_like(x.shape, x.dtype)
    dx3 = dx.view(B, S, D)
    per_sample = g.mod_stride != 0
    sc = scale.to(dev, non_blocking=True).to(x.dtype)
    flag = torch.zeros(1, dtype=torch.int32, device=dev) if check_finite else None
    main, side = torch.cuda.current_stream(dev), _side(dev)
    xres = _resident.get(x, dev)  # the forward's device copy of this x, if still valid
    parts = []  # (b0, b1, dscale chunk, dshift chunk) on the device
    # chunks sized by the bytes that actually move in (dy, and x unless it is resident)
    in_row = (1 if xres is not None else 2) * D * x.element_size()
    for b0, b1, s0, s1 in _chunks(B, S, in_row):
        xd = xres[b0:b1, s0:s1] if xres is not None else x3[b0:b1, s0:s1].to(dev, non_blocking=True)
        dyd = dy3[b0:b1, s0:s1].to(dev, non_blocking=True)
        mud = mu2[b0:b1, s0:s1].to(dev, non_blocking=True)
        rsd = rs2[b0:b1, s0:s1].to(dev, non_blocking=True)
        scb = sc[b0:b1] if per_sample else sc
        nt = min(n_tile, (s1 - s0) if per_sample else (b1 - b0) * (s1 - s0)) if n_tile else 0
        dxd, dsc, dsh = fused_backward(dyd, xd, scb, mud, rsd, d_tile=d_tile if nt else 0,
                                       n_tile=nt, flag=flag, deterministic=True)
        parts.append((b0, b1, dsc, dsh))
        side.wait_stream(main)
        with torch.cuda.stream(side):
            dx3[b0:b1, s0:s1].copy_(dxd, non_blocking=True)
        for t in (dyd, mud, rsd, dxd) if xres is not None else (xd, dyd, mud, rsd, dxd):
            t.record_stream(side)
    # fixed-order fp64 sum of the chunk partials
    acc_sc = torch.zeros((B, D) if per_sample else (D,), dtype=torch.float64, device=dev)
    acc_sh = torch.zeros_like(acc_sc)
    for b0, b1, dsc, dsh in parts:
        if per_sample:
            acc_sc[b0:b1] += dsc.double()
            acc_sh[b0:b1] += dsh.double()
        else:
            acc_sc += dsc.double()
            acc_sh += dsh.double()
    dscale = acc_sc.to(sdt).cpu()
    dshift = acc_sh.to(sdt).cpu()
    side.synchronize()
    if flag is not None and int(flag.item()):
        raise NonFiniteInput("dy/x/scale contains NaN or Inf")
    return dx, dscale, dshift
