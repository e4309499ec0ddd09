"""Slab-decomposed distributed 2D/3D FFTs on B200 (drop-in for distfft.py).

Reference: /root/reference/pkg/src/pfcspectral/distfft.py:1-209.  Same
layouts, same public functions and the same errors; the local slab of a
:class:`DistField` lives on the worker's GPU (``field.dev``) and
``field.local`` is a host (numpy) view materialised on access.

3D pipeline (distfft.py:150-173), physical Z_SLAB (nx, ny, cz) <-> spectral
X_SLAB (cx, ny, nz):

    forward : x-lines (strided)  -> y-lines (strided)  -> all-to-all
              -> z-lines reading the receive buffer directly (the
                 reference's np.concatenate along z, distfft.py:120, is the
                 kernel's gather addressing)
    inverse : z-lines writing straight into per-destination send blocks
              -> all-to-all -> x-lines -> y-lines

Because x is the slowest axis, the forward send blocks are contiguous row
ranges (no pack kernel) and the inverse receive buffer *is* the Z slab (no
unpack kernel): the exchange costs zero extra HBM passes.

2D (nz == 1, distfft.py:176-195) runs the identical pipeline on the
(nx, 1, ny) view of the array: Y_SLAB (nx, cy, 1) and X_SLAB (cx, ny, 1) are
byte-identical to Z_SLAB/X_SLAB of that view.

Real fields (float64 ``local``) take the R2C/C2R path: the x pass packs the
real line into a half-length complex FFT and keeps nx/2+1 modes, the
spectral X slab splits those nx/2+1 modes over the ranks.  Complex fields
(the reference's complex128 convention) take the C2C path.
"""

from __future__ import annotations

import enum

import warnings

import numpy as np
import torch

from . import _native as nat
from .grid import GridSpec, SlabLayout, slab_layout

__all__ = [
    "Layout",
    "Space",
    "DistField",
    "layout_for",
    "scatter",
    "gather",
    "exchange_z_to_x",
    "exchange_x_to_z",
    "exchange_y_to_x",
    "exchange_x_to_y",
    "dist_fft_forward",
    "dist_fft_inverse",
    "dist_fft_2d_forward",
    "dist_fft_2d_inverse",
    "forward",
    "inverse",
    "physical_layout",
    "half_modes",
]


class Layout(enum.Enum):
    Z_SLAB = 2  # value doubles as the decomposition axis (distfft.py:48-51)
    X_SLAB = 0
    Y_SLAB = 1


class Space(enum.Enum):
    PHYSICAL = "physical"
    SPECTRAL = "spectral"


def half_modes(grid: GridSpec) -> int:
    """Number of x modes kept by the real-to-complex transform."""
    return grid.n[0] // 2 + 1


def _device_of(worker) -> torch.device:
    dev = getattr(worker, "device", None) if worker is not None else None
    if dev is None:
        nat.load()
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


class DistField:
    """One worker's slab of a distributed field (distfft.py:59-72).

    ``dev``   : the slab on the GPU (complex128, or float64 for a real
                physical field); C-order in the reference's local shape.
    ``local`` : numpy copy of ``dev`` (reading it synchronises); assigning
                an array uploads it.
    ``half``  : spectral data holding only the nx/2+1 non-negative x modes
                of a real field (R2C representation).
    """

    def __init__(self, grid: GridSpec, layout: Layout, space: Space, local, *, half: bool = False,
                 device=None):
        self.grid = grid
        self.layout = layout
        self.space = space
        self.half = bool(half)
        self._version = 0
        self._device = device
        self._dev = None
        self._set(local)

    def _set(self, data) -> None:
        if isinstance(data, torch.Tensor):
            if not data.is_cuda:
                nat.load()
                data = data.to(self._device or torch.device("cuda", torch.cuda.current_device()))
            t = data.contiguous()
        else:
            arr = np.asarray(data)
            if arr.dtype not in (np.float64, np.complex128):
                arr = arr.astype(np.complex128)
            nat.load()
            dev = self._device or torch.device("cuda", torch.cuda.current_device())
            t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        self._dev = t
        self._device = t.device
        self._version += 1

    @property
    def dev(self) -> torch.Tensor:
        return self._dev

    @dev.setter
    def dev(self, t: torch.Tensor) -> None:
        self._set(t)

    @property
    def local(self) -> np.ndarray:
        """Read-only host copy of the slab: in-place edits of the copy would
        not reach the device, so they fail loudly instead of being lost
        (assign ``field.local = array`` to upload).  Code that edits
        ``field.dev`` in place must call :meth:`touch` so cached work derived
        from the field (the PFC engine's prepared inverse) is rebuilt."""
        a = self._dev.cpu().numpy()
        a.setflags(write=False)
        return a

    def touch(self) -> None:
        """Mark the device slab as modified in place (bumps the version)."""
        self._version += 1

    @local.setter
    def local(self, value) -> None:
        self._set(value)

    @property
    def is_real(self) -> bool:
        return not self._dev.is_complex()

    def expected_shape(self, rank: int, workers: int) -> tuple[int, int, int]:
        lay = _layout(self.grid, self.layout, workers, self.half)
        shape = list(self.grid.shape)
        if self.half:
            shape[0] = half_modes(self.grid)
        shape[lay.axis] = lay.counts[rank]
        return tuple(shape)


def layout_for(grid: GridSpec, layout: Layout, workers: int) -> SlabLayout:
    """Balanced slab layout of ``layout``'s split axis (distfft.py:75-77)."""
    axis = layout.value
    return slab_layout(grid.n[axis], workers, axis=axis)


def _layout(grid: GridSpec, layout: Layout, workers: int, half: bool) -> SlabLayout:
    if half and layout is Layout.X_SLAB:
        return slab_layout(half_modes(grid), workers, axis=0)
    return layout_for(grid, layout, workers)


def physical_layout(grid: GridSpec) -> Layout:
    """Z slabs in 3D, Y slabs in 2D (distfft.py:80-82)."""
    return Layout.Y_SLAB if grid.is_2d else Layout.Z_SLAB


def _local_slice(lay: SlabLayout, rank: int) -> tuple:
    sl = [slice(None)] * 3
    sl[lay.axis] = lay.local_slice(rank)
    return tuple(sl)


def scatter(full, worker, grid: GridSpec, layout: Layout, space: Space = Space.PHYSICAL,
            *, real: bool = False) -> DistField:
    """This worker's slab of a replicated full array (distfft.py:91-100).

    As in the reference the slab is cast to complex128; ``real=True`` keeps a
    float64 physical slab, which routes the transforms through R2C/C2R."""
    if tuple(full.shape) != grid.shape:
        raise ValueError(f"scatter: array shape {full.shape} does not match grid {grid.shape}")
    lay = layout_for(grid, layout, worker.size)
    dtype = np.float64 if real else np.complex128
    if real and np.iscomplexobj(full):
        raise ValueError("scatter(real=True) needs a real array")
    part = np.ascontiguousarray(np.asarray(full)[_local_slice(lay, worker.rank)], dtype=dtype)
    return DistField(grid, layout, space, part, device=_device_of(worker))


def _expand_half(half: np.ndarray, nx: int) -> np.ndarray:
    """Full spectrum of a real field from its nx/2+1 x modes (Hermitian
    symmetry X[-k] = conj X[k])."""
    full = np.empty((nx,) + half.shape[1:], dtype=np.complex128)
    m = half.shape[0]
    full[:m] = half
    if nx > m:
        src = half[1:nx - m + 1][::-1]  # modes nx-m .. 1 mirrored
        idx_y = (-np.arange(half.shape[1])) % half.shape[1]
        idx_z = (-np.arange(half.shape[2])) % half.shape[2]
        full[m:] = np.conj(src[:, idx_y][:, :, idx_z])
    return full


def gather(field: DistField, worker) -> np.ndarray:
    """Reassemble the full array on every rank (distfft.py:103-107).  A
    half-spectrum field is returned as the full (Hermitian) spectrum."""
    if not isinstance(field.layout, Layout):
        from .pencil import pencil_gather

        return pencil_gather(field, worker)
    received = worker.all_to_all([field.local] * worker.size)
    lay = _layout(field.grid, field.layout, worker.size, field.half)
    full = np.concatenate(received, axis=lay.axis)
    if field.half:
        full = _expand_half(full, field.grid.n[0])
    return full


# ------------------------------------------------------------------ views ----

def _dims3(grid: GridSpec) -> tuple[int, int, int]:
    """(nx, ny, nz) of the 3D view the kernels run on: 2D grids are viewed as
    (nx, 1, ny) so the y-slab pipeline is the z-slab pipeline."""
    nx, ny, nz = grid.n
    return (nx, 1, ny) if nz == 1 else (nx, ny, nz)


def _counts(n: int, G: int) -> list[int]:
    return list(slab_layout(n, G).counts)


class _Geometry:
    """Per-(grid, G, rank, real) slab sizes of the (nx', ny', nz') view."""

    def __init__(self, grid: GridSpec, G: int, rank: int, real: bool):
        self.nx, self.ny, self.nz = _dims3(grid)
        self.G, self.rank, self.real = G, rank, real
        self.nxm = self.nx // 2 + 1 if real else self.nx  # x modes on the spectral side
        self.cx_all = _counts(self.nxm, G)
        self.cz_all = _counts(self.nz, G)
        self.cx = self.cx_all[rank]
        self.cz = self.cz_all[rank]
        self.xoff = sum(self.cx_all[:rank])

    # forward exchange: send rows of the (nxm, ny, cz) slab, receive blocked z
    def fwd_counts(self):
        send = [c * self.ny * self.cz for c in self.cx_all]
        recv = [self.cx * self.ny * c for c in self.cz_all]
        return send, recv

    def inv_counts(self):
        recv, send = self.fwd_counts()
        return send, recv

    @property
    def zslab_elems(self) -> int:
        return self.nxm * self.ny * self.cz

    @property
    def xslab_elems(self) -> int:
        return self.cx * self.ny * self.nz


def _stream() -> int:
    return nat.stream_ptr()


def _fft_x(t: torch.Tensor, g: _Geometry, forward: bool, out: torch.Tensor) -> None:
    """C2C x-lines of an (nx, ny, cz) complex slab."""
    nat.call("pfcs_fft_axis_c2c", nat.ptr(t), nat.ptr(out), g.nx, g.ny, g.cz, 0,
             1 if forward else 0, _stream())


def _fft_y(t: torch.Tensor, g: _Geometry, forward: bool) -> None:
    """y-lines in place on an (nxm, ny, cz) complex slab."""
    if g.ny > 1:
        nat.call("pfcs_fft_axis_c2c", nat.ptr(t), nat.ptr(t), g.nxm, g.ny, g.cz, 1,
                 1 if forward else 0, _stream())


def _ensure(field: DistField, layout: Layout, space: Space) -> None:
    if field.layout is not layout or field.space is not space:
        raise ValueError(f"expected {layout.name}/{space.name} field, "
                         f"got {field.layout.name}/{field.space.name}")


class _PeerPlan:
    """Receive buffers of one (grid, G, real) slab pipeline mapped on every
    rank, for the fused exchanges (see peer.py)."""

    def __init__(self, worker, g: "_Geometry"):
        from . import peer

        self.bz = peer.DeviceBuffer(g.zslab_elems)
        self.bx = peer.DeviceBuffer(g.xslab_elems)
        mz = peer.map_peers(worker, self.bz)
        mx = peer.map_peers(worker, self.bx)
        self.maps = (mz, mx)
        zoff = [sum(g.cz_all[:h]) for h in range(g.G)]
        self.tab_z = peer.Table([mz.addrs[h] + 16 * g.xoff * g.ny * g.cz_all[h] for h in range(g.G)])
        self.tab_x = peer.Table([mx.addrs[h] + 16 * g.cx_all[h] * g.ny * zoff[g.rank] for h in range(g.G)])


def _pow2(n: int) -> bool:
    return n >= 2 and (n & (n - 1)) == 0


def _peer_plan(worker, g: "_Geometry"):
    """Fused-exchange plan for this pipeline, or None (collective path):
    needs G > 1, a y axis to carry the forward scatter and power-of-two
    y/z lines <= 4096 (PFCS_EXCHANGE=collective disables it)."""
    from .pfc import exchange_mode

    if g.G == 1 or g.ny < 2 or not (_pow2(g.ny) and _pow2(g.nz)) or exchange_mode() != "peer":
        return None
    if g.ny > 4096 or g.nz > 4096:  # the fused scatter kernels' Stockham lengths
        return None
    if min(g.cz_all) < 2:  # the y-line scatter tiles need >= 2 contiguous z columns
        return None
    plans = worker.__dict__.setdefault("_pfcs_plans", {})
    key = (g.nx, g.ny, g.nz, g.real)
    if key not in plans:
        from .peer import PeerUnavailable

        try:
            plans[key] = _PeerPlan(worker, g)
        except PeerUnavailable as exc:  # every rank: the collective path from now on
            warnings.warn(f"fused peer exchange unavailable ({exc}); using the collective all-to-all")
            plans[key] = None
    return plans[key]


def _forward_core(src: torch.Tensor, worker, g: _Geometry) -> torch.Tensor:
    """Physical Z slab (flat) -> spectral X slab (flat, plain layout)."""
    dev = src.device
    a = torch.empty(g.zslab_elems, dtype=torch.complex128, device=dev)
    if g.real:
        nat.call("pfcs_rfft_x", nat.ptr(src), nat.ptr(a), g.nx, g.ny * g.cz, _stream())
    else:
        _fft_x(src, g, True, a)
    plan = _peer_plan(worker, g)
    if plan is not None:
        # y lines stored straight into the owners' blocked-z receive buffers
        from .peer import fence

        fence(worker)  # every rank is done reading its buffer from the last call
        nat.call("pfcs_fft_lines_scatter", nat.ptr(a), plan.tab_x.ptr, g.nxm, g.ny, g.cz, 1, g.G, 1, _stream())
        fence(worker)
        out = torch.empty(g.xslab_elems, dtype=torch.complex128, device=dev)
        nat.call("pfcs_fft_zlines", nat.ptr(plan.bx.tensor), nat.ptr(out), g.cx * g.ny, g.nz, g.G, 1, 1,
                 _stream())
        return out
    _fft_y(a, g, True)
    if g.G == 1:
        nat.call("pfcs_fft_zlines", nat.ptr(a), nat.ptr(a), g.cx * g.ny, g.nz, 1, 1, 1, _stream())
        return a
    recv = torch.empty(g.xslab_elems, dtype=torch.complex128, device=dev)
    sc, rc = g.fwd_counts()
    worker.exchange(a, sc, recv, rc)
    out = torch.empty(g.xslab_elems, dtype=torch.complex128, device=dev)
    nat.call("pfcs_fft_zlines", nat.ptr(recv), nat.ptr(out), g.cx * g.ny, g.nz, g.G, 1, 1, _stream())
    return out


def _inverse_core(src: torch.Tensor, worker, g: _Geometry) -> torch.Tensor:
    """Spectral X slab (flat, plain) -> physical Z slab (flat)."""
    dev = src.device
    plan = _peer_plan(worker, g)
    if plan is not None:
        # z lines stored straight into the owners' Z-slab receive buffers
        from .peer import fence

        fence(worker)
        nat.call("pfcs_fft_zlines_to", nat.ptr(src), plan.tab_z.ptr, g.cx * g.ny, g.nz, 1, g.G, 0, _stream())
        fence(worker)
        z = plan.bz.tensor[:g.zslab_elems]
        _fft_y(z, g, False)
        if g.real:
            out = torch.empty(g.nx * g.ny * g.cz, dtype=torch.float64, device=dev)
            nat.call("pfcs_irfft_x", nat.ptr(z), nat.ptr(out), g.nx, g.ny * g.cz, _stream())
            return out
        out = torch.empty(g.zslab_elems, dtype=torch.complex128, device=dev)
        _fft_x(z, g, False, out)
        return out
    send = torch.empty(g.xslab_elems, dtype=torch.complex128, device=dev)
    nat.call("pfcs_fft_zlines", nat.ptr(src), nat.ptr(send), g.cx * g.ny, g.nz, 1, g.G, 0, _stream())
    if g.G == 1:
        z = send
    else:
        z = torch.empty(g.zslab_elems, dtype=torch.complex128, device=dev)
        sc, rc = g.inv_counts()
        worker.exchange(send, sc, z, rc)
    if g.real:
        _fft_y(z, g, False)
        out = torch.empty(g.nx * g.ny * g.cz, dtype=torch.float64, device=dev)
        nat.call("pfcs_irfft_x", nat.ptr(z), nat.ptr(out), g.nx, g.ny * g.cz, _stream())
        return out
    # y then x, the order of the fused PFC step (so distfft.inverse and the
    # stepper's internal psi are bit-identical)
    _fft_y(z, g, False)
    _fft_x(z, g, False, z)
    return z


def _check_real_support(grid: GridSpec) -> None:
    nx = grid.n[0]
    if nx < 4 or nx & (nx - 1):
        raise ValueError(f"real-to-complex transforms need a power-of-two nx >= 4, got {nx}")


def _forward(field: DistField, worker, phys: Layout) -> DistField:
    _ensure(field, phys, Space.PHYSICAL)
    real = field.is_real
    if real:
        _check_real_support(field.grid)
    g = _Geometry(field.grid, worker.size, worker.rank, real)
    src = field.dev.reshape(-1)
    out = _forward_core(src, worker, g)
    if worker.meter is not None:
        worker.meter.sample(src.numel() * src.element_size() + 2 * out.numel() * 16)
    nx, ny, nz = field.grid.n
    shape = (g.cx, ny, nz)
    return DistField(field.grid, Layout.X_SLAB, Space.SPECTRAL, out.view(shape), half=real,
                     device=out.device)


def _inverse(field: DistField, worker, phys: Layout) -> DistField:
    _ensure(field, Layout.X_SLAB, Space.SPECTRAL)
    real = field.half
    g = _Geometry(field.grid, worker.size, worker.rank, real)
    src = field.dev.reshape(-1)
    if not src.is_complex():
        raise ValueError("spectral fields must be complex")
    out = _inverse_core(src, worker, g)
    if worker.meter is not None:
        worker.meter.sample(src.numel() * 16 + 2 * out.numel() * out.element_size())
    nx, ny, nz = field.grid.n
    shape = (nx, ny, g.cz) if nz > 1 else (nx, g.cz, 1)
    return DistField(field.grid, phys, Space.PHYSICAL, out.view(shape), device=out.device)


def dist_fft_forward(field: DistField, worker) -> DistField:
    """Z-slab physical -> X-slab spectral (distfft.py:150-160)."""
    return _forward(field, worker, Layout.Z_SLAB)


def dist_fft_inverse(field: DistField, worker) -> DistField:
    """X-slab spectral -> Z-slab physical (distfft.py:163-173)."""
    return _inverse(field, worker, Layout.Z_SLAB)


def dist_fft_2d_forward(field: DistField, worker) -> DistField:
    """Y-slab physical -> X-slab spectral, nz == 1 (distfft.py:176-184)."""
    return _forward(field, worker, Layout.Y_SLAB)


def dist_fft_2d_inverse(field: DistField, worker) -> DistField:
    """X-slab spectral -> Y-slab physical, nz == 1 (distfft.py:187-195)."""
    return _inverse(field, worker, Layout.Y_SLAB)


def forward(field: DistField, worker) -> DistField:
    """Dimension-dispatching forward transform (distfft.py:198-202); pencil
    layouts (pencil.PencilLayout) take the pencil pipeline."""
    if not isinstance(field.layout, Layout):
        from .pencil import pencil_forward

        return pencil_forward(field, worker)
    if field.grid.is_2d:
        return dist_fft_2d_forward(field, worker)
    return dist_fft_forward(field, worker)


def inverse(field: DistField, worker) -> DistField:
    """Dimension-dispatching inverse transform (distfft.py:205-209); pencil
    layouts take the pencil pipeline."""
    if not isinstance(field.layout, Layout):
        from .pencil import pencil_inverse

        return pencil_inverse(field, worker)
    if field.grid.is_2d:
        return dist_fft_2d_inverse(field, worker)
    return dist_fft_inverse(field, worker)


# --------------------------------------------------------------- exchanges ---

def _exchange(field: DistField, worker, src_layout: Layout, dst_layout: Layout) -> DistField:
    """Pure data movement between slab layouts (distfft.py:110-124): every
    block goes to its owner, received blocks are concatenated along the
    source split axis.  Runs as one device all-to-all plus a strided copy
    into the destination layout."""
    if field.layout is not src_layout:
        raise ValueError(f"exchange expects {src_layout.name} input, got {field.layout.name}")
    G = worker.size
    grid = field.grid
    src_lay = _layout(grid, src_layout, G, field.half)
    dst_lay = _layout(grid, dst_layout, G, field.half)
    t = field.dev
    shape = list(t.shape)
    # blocks of the local slab destined to each rank: slices along dst axis
    blocks = [t.narrow(dst_lay.axis, dst_lay.offsets[h], dst_lay.counts[h]).contiguous().reshape(-1)
              for h in range(G)]
    send = torch.cat(blocks) if G > 1 else blocks[0]
    send_counts = [b.numel() for b in blocks]
    out_shape = list(shape)
    out_shape[dst_lay.axis] = dst_lay.counts[worker.rank]
    out_shape[src_lay.axis] = grid.n[src_lay.axis] if not (field.half and src_lay.axis == 0) \
        else half_modes(grid)
    recv_counts = []
    for g in range(G):
        s = list(out_shape)
        s[src_lay.axis] = src_lay.counts[g]
        recv_counts.append(int(np.prod(s)))
    recv = torch.empty(sum(recv_counts), dtype=t.dtype, device=t.device)
    worker.exchange(send, send_counts, recv, recv_counts)
    parts = []
    off = 0
    for g in range(G):
        s = list(out_shape)
        s[src_lay.axis] = src_lay.counts[g]
        parts.append(recv[off:off + recv_counts[g]].view(s))
        off += recv_counts[g]
    local = torch.cat(parts, dim=src_lay.axis).contiguous() if G > 1 else parts[0].clone()
    if worker.meter is not None:
        worker.meter.sample(t.numel() * t.element_size() + local.numel() * local.element_size())
    return DistField(grid, dst_layout, field.space, local, half=field.half, device=local.device)


def exchange_z_to_x(field: DistField, worker) -> DistField:
    return _exchange(field, worker, Layout.Z_SLAB, Layout.X_SLAB)


def exchange_x_to_z(field: DistField, worker) -> DistField:
    return _exchange(field, worker, Layout.X_SLAB, Layout.Z_SLAB)


def exchange_y_to_x(field: DistField, worker) -> DistField:
    return _exchange(field, worker, Layout.Y_SLAB, Layout.X_SLAB)


def exchange_x_to_y(field: DistField, worker) -> DistField:
    return _exchange(field, worker, Layout.X_SLAB, Layout.Y_SLAB)
