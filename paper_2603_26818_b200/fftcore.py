"""Serial complex-to-complex FFTs on B200 (drop-in for fftcore.py).

Reference: /root/reference/pkg/src/pfcspectral/fftcore.py:1-52.  Same
conventions: forward unnormalised, inverse scaled by fl(1/n) per axis;
length-1 axes copy, empty arrays return empty copies.  The multi-axis order
is pinned — forward 0,1,2 and inverse 2,1,0 — so that, as in the reference
(fftcore.py:4-11, which pins 2,0,1 for the same purpose), the serial
transform, the distributed one and the fused PFC pipeline (z, y, then x
innermost) follow bit-identical arithmetic; e.g. the hydro density update
with v = 0 reproduces pfc_step bit for bit.

Arrays may be numpy arrays (the reference's type — they are moved to the
current CUDA device and the result comes back as numpy) or CUDA tensors
(stay on the device: the hot path used by the hydro solver).  The
arithmetic always runs in libpfcs (no CPU fallback).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat

__all__ = ["fft_axis", "fft_2d", "fft_nd"]


def _check(shape, axis: int) -> None:
    if len(shape) != 3:
        raise ValueError(f"expected a 3D buffer, got shape {tuple(shape)}")
    if axis not in (0, 1, 2):
        raise ValueError(f"axis must be 0, 1 or 2, got {axis}")


def _to_device(a) -> tuple[torch.Tensor, bool]:
    if isinstance(a, torch.Tensor):
        t = a if a.is_complex() else a.to(torch.complex128)
        if t.dtype != torch.complex128:
            t = t.to(torch.complex128)
        if not t.is_cuda:
            nat.load()
            t = t.cuda()
        return t.contiguous(), False
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
    nat.load()
    return torch.from_numpy(arr).to(torch.device("cuda", torch.cuda.current_device())), True


def _axis_inplace(t: torch.Tensor, axis: int, forward: bool, out: torch.Tensor) -> None:
    n0, n1, n2 = t.shape
    nat.call("pfcs_fft_axis_c2c", nat.ptr(t), nat.ptr(out), n0, n1, n2, axis, 1 if forward else 0,
             nat.stream_ptr())


def fft_axis(a, axis: int, forward: bool = True):
    """1D DFT along one axis of a 3D complex buffer (fftcore.py:31-40)."""
    _check(a.shape, axis)
    t, host = _to_device(a)
    out = torch.empty_like(t)
    if t.numel():
        _axis_inplace(t, axis, forward, out)
    return out.cpu().numpy() if host else out


def fft_2d(a, forward: bool = True):
    """Axes 0 and 1, every z-plane independently: axis 0 then axis 1 in
    both directions, the reference's composition (fftcore.py:43-45)."""
    _check(a.shape, 0)
    t, host = _to_device(a)
    out = torch.empty_like(t)
    if t.numel():
        _axis_inplace(t, 0, forward, out)
        _axis_inplace(out, 1, forward, out)
    return out.cpu().numpy() if host else out


def fft_nd(a, forward: bool = True):
    """All axes; forward 0,1,2 and inverse 2,1,0 (fftcore.py:48-52)."""
    _check(a.shape, 0)
    t, host = _to_device(a)
    out = torch.empty_like(t)
    if t.numel():
        order = (0, 1, 2) if forward else (2, 1, 0)
        _axis_inplace(t, order[0], forward, out)
        for ax in order[1:]:
            _axis_inplace(out, ax, forward, out)
    return out.cpu().numpy() if host else out
