"""Semi-implicit pseudo-spectral PFC solver on B200 (drop-in for pfc.py).

Reference: /root/reference/pkg/src/pfcspectral/pfc.py:1-310.

    psi_hat <- (psi_hat + dt * lap * F[psi^3]) / (1 - dt * lin)

One step (pfc.py:96-128) is an inverse transform, a pointwise cube, a
forward transform and the implicit update.  Here the step is five fused
device passes on the worker's slab (R2C representation shown; C2C is the
same with full x lines):

    K_y^-1   y-lines inverse                        (receive buffer, in place)
    K_x      x-lines: C2R -> psi^3 -> R2C, plus max|psi| diagnostics
    K_y      y-lines forward                        (in place)
    --- all-to-all (NCCL / NVLink) ---
    K_z      z-lines: forward FFT (reads the receive blocks) -> implicit
             update of psi_hat -> finiteness flag -> inverse FFT of the new
             psi_hat written into the next step's send blocks
    --- all-to-all ---

so each step moves 10 half-spectrum volumes through HBM
and the physical field never leaves shared memory.  Grids the fused passes
do not cover (non-power-of-two axes) take an unfused sequence of the same
kernels' building blocks with identical update arithmetic.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, field as dataclass_field

import numpy as np
import torch

from . import _native as nat
from . import distfft
from .distfft import DistField, Layout, Space, _Geometry
from .grid import GridSpec, SymbolTable, wavenumbers

__all__ = [
    "PfcParams",
    "PfcState",
    "DivergenceError",
    "IncommensurateDomainError",
    "pfc_step",
    "pfc_run",
    "free_energy",
    "mean_and_max",
    "initial_field",
    "init_condition",
    "default_domain_length",
    "TRIANGULAR_Q",
    "FCC_Q1",
    "INIT_KINDS",
    "initial_field_slab",
]

# lattice wavenumbers on the zeros of the two-ring symbol (pfc.py:43-46)
TRIANGULAR_Q = math.sqrt(3.0) / 2.0
FCC_Q1 = 1.0 / math.sqrt(3.0)

INIT_KINDS = (
    "constant_plus_noise",
    "seeded_crystallites",
    "single_mode_triangular_2d",
    "two_mode_fcc_3d",
)


class DivergenceError(RuntimeError):
    """Non-finite field at ``step_index`` (pfc.py:53-58)."""

    def __init__(self, step_index: int, max_abs: float):
        super().__init__(f"non-finite field at step {step_index} (max |psi| = {max_abs:g})")
        self.step_index = step_index
        self.max_abs = max_abs


class IncommensurateDomainError(ValueError):
    pass


@dataclass
class PfcParams:
    eps: float = -0.3
    dt: float = 0.1
    psi_bar: float = -0.3
    n_steps: int = 100

    def __post_init__(self):
        if not all(math.isfinite(v) for v in (self.eps, self.dt, self.psi_bar)):
            raise ValueError("PfcParams fields must be finite")
        if self.dt <= 0:
            raise ValueError(f"dt must be positive, got {self.dt}")
        if self.n_steps < 0:
            raise ValueError(f"n_steps must be >= 0, got {self.n_steps}")


@dataclass
class PfcState:
    """Per-worker solver state; ``psi_hat`` is an X-slab spectral field
    (pfc.py:82-93).  ``_engine`` holds device workspaces and the cached
    first stage of the next inverse transform."""

    psi_hat: DistField
    grid: GridSpec
    symbols: SymbolTable
    worker: object
    step_index: int = 0
    sim_time: float = 0.0
    last_max_imag_ratio: float = dataclass_field(default=0.0)
    _engine: object = dataclass_field(default=None, repr=False, compare=False)


def _pow2(n: int) -> bool:
    return n >= 2 and (n & (n - 1)) == 0


def exchange_mode() -> str:
    """'peer' (default): transposes fused into the FFT epilogues, stores to
    peer-mapped receive buffers; 'collective': separate all-to-all
    (NCCL all_to_all_single / device copies).  PFCS_EXCHANGE overrides."""
    import os

    mode = os.environ.get("PFCS_EXCHANGE", "peer").lower()
    if mode not in ("peer", "collective"):
        raise ValueError(f"PFCS_EXCHANGE must be 'peer' or 'collective', got {mode!r}")
    return mode


class _StepEngine:
    """Workspaces and launch sequence of one rank's PFC step."""

    def __init__(self, state: PfcState):
        f = state.psi_hat
        self.real = f.half
        self.grid = state.grid
        self.worker = state.worker
        self.G = self.worker.size
        self.rank = self.worker.rank
        self.g = _Geometry(state.grid, self.G, self.rank, self.real)
        g = self.g
        self.device = f.dev.device
        nx3, ny3, nz3 = g.nx, g.ny, g.nz
        # fused passes need power-of-two x (>= 4 real, >= 2 complex) and z
        self.fused = _pow2(nz3) and nz3 <= 4096 and (
            (self.real and _pow2(nx3) and 4 <= nx3 <= 8192) or
            (not self.real and _pow2(nx3) and nx3 <= 4096))
        cdt = torch.complex128
        self.peer = False
        if self.G == 1:
            self.work = torch.empty(max(g.zslab_elems, 1), dtype=cdt, device=self.device)
            self.send = self.recv_z = self.recv_x = self.work
        elif (self.fused and g.ny > 1 and _pow2(g.ny) and g.ny <= 4096 and min(g.cz_all) > 1
              and exchange_mode() == "peer"):
            # the fused y-line scatter (pfcs_fft_lines_scatter) needs
            # power-of-two y lines <= 4096; other y extents take the collective
            from .peer import PeerUnavailable

            try:
                self._setup_peer()
            except PeerUnavailable as exc:  # on every rank: collective buffers instead
                warnings.warn(f"fused peer exchange unavailable ({exc}); using the collective all-to-all")
                self._bz = self._bx = self._maps = None
        if not self.peer and self.G > 1:
            self.send = torch.empty(max(g.xslab_elems, 1), dtype=cdt, device=self.device)
            self.recv_z = torch.empty(max(g.zslab_elems, 1), dtype=cdt, device=self.device)
            self.recv_x = torch.empty(max(g.xslab_elems, 1), dtype=cdt, device=self.device)
        self.diag = torch.zeros(nat.DIAG_SLOTS * nat.DIAG_VALS, dtype=torch.float64, device=self.device)
        self.kvec = None
        self.prepared_for = None  # (id(tensor), version) the send buffer was built from

    def _setup_peer(self) -> None:
        """Fused exchanges: the receive buffers are mapped on every rank and
        the kernels before each transpose store into them directly (collective:
        all ranks build their engine in the same step)."""
        from . import peer

        g, G, me = self.g, self.G, self.rank
        self._bz = peer.DeviceBuffer(g.zslab_elems, device=self.device)
        self._bx = peer.DeviceBuffer(g.xslab_elems, device=self.device)
        mz = peer.map_peers(self.worker, self._bz)
        mx = peer.map_peers(self.worker, self._bx)
        self._maps = (mz, mx)
        self.recv_z, self.recv_x = self._bz.tensor, self._bx.tensor
        self.send = None
        zoff = [sum(g.cz_all[:h]) for h in range(G)]
        # my z-inverse block for rank h lands at rows xoff..xoff+cx of its Z slab
        self.tab_z = peer.Table([mz.addrs[h] + 16 * g.xoff * g.ny * g.cz_all[h] for h in range(G)])
        # my y-forward rows for rank h land in its blocked-z buffer, block `me`
        self.tab_x = peer.Table([mx.addrs[h] + 16 * g.cx_all[h] * g.ny * zoff[me] for h in range(G)])
        self.peer = True

    def _sym_ptrs(self, sym):
        if self.kvec is None or self.kvec[0] is not sym:
            self.kvec = (sym, slab_kvectors(self.grid, sym, self.g, self.device))
        kx, ky, kz = self.kvec[1]
        return nat.ptr(kx), nat.ptr(ky), nat.ptr(kz)

    def invalidate(self) -> None:
        self.prepared_for = None

    def launch(self, state: PfcState, params: PfcParams, diag: torch.Tensor) -> None:
        """Enqueue one step on the current stream (no host synchronisation);
        ``diag`` (zeroed) receives the step's diagnostics."""
        g = self.g
        st = nat.stream_ptr()
        psi = state.psi_hat.dev
        if psi.dtype != torch.complex128 or not psi.is_contiguous():
            raise ValueError("psi_hat must be a contiguous complex128 slab")
        kx, ky, kz = self._sym_ptrs(state.symbols)
        dptr = nat.ptr(diag)
        key = (psi.data_ptr(), state.psi_hat._version)
        nlines = g.cx * g.ny
        eps, dt = float(state.symbols.eps), float(params.dt)
        if self.peer:
            # fused exchanges: K_z and K_y store straight into the owners'
            # receive buffers (NVLink peer / IPC), a fence orders each transpose
            from .peer import fence

            if self.prepared_for != key:
                nat.call("pfcs_fft_zlines_to", nat.ptr(psi), self.tab_z.ptr, nlines, g.nz, 1, self.G, 0, st)
                fence(self.worker)
            z = self.recv_z
            nat.call("pfcs_fft_axis_c2c", nat.ptr(z), nat.ptr(z), g.nxm, g.ny, g.cz, 1, 0, st)
            nat.call("pfcs_pfc_cube_x", nat.ptr(z), g.nx, g.ny * g.cz, 1 if self.real else 0, dptr, st)
            nat.call("pfcs_fft_lines_scatter", nat.ptr(z), self.tab_x.ptr, g.nxm, g.ny, g.cz, 1, self.G, 1, st)
            fence(self.worker)
            nat.call("pfcs_pfc_update_z_to", nat.ptr(self.recv_x), nat.ptr(psi), self.tab_z.ptr, g.cx, g.ny,
                     g.nz, self.G, self.G, kx, ky, kz, eps, dt, dptr, st)
            fence(self.worker)
        elif self.fused:
            if self.prepared_for != key:
                nat.call("pfcs_fft_zlines", nat.ptr(psi), nat.ptr(self.send), nlines, g.nz, 1, self.G, 0, st)
            if self.G > 1:
                sc, rc = g.inv_counts()
                self.worker.exchange(self.send, sc, self.recv_z, rc)
            z = self.recv_z
            if g.ny > 1:
                nat.call("pfcs_fft_axis_c2c", nat.ptr(z), nat.ptr(z), g.nxm, g.ny, g.cz, 1, 0, st)
            nat.call("pfcs_pfc_cube_x", nat.ptr(z), g.nx, g.ny * g.cz, 1 if self.real else 0, dptr, st)
            if g.ny > 1:
                nat.call("pfcs_fft_axis_c2c", nat.ptr(z), nat.ptr(z), g.nxm, g.ny, g.cz, 1, 1, st)
            if self.G > 1:
                sc, rc = g.fwd_counts()
                self.worker.exchange(z, sc, self.recv_x, rc)
            nat.call("pfcs_pfc_update_z", nat.ptr(self.recv_x), nat.ptr(psi), nat.ptr(self.send),
                     g.cx, g.ny, g.nz, self.G, self.G, kx, ky, kz, eps, dt, dptr, st)
        else:
            self._unfused(state, params, kx, ky, kz, dptr, st)
        state.psi_hat._version += 1
        self.prepared_for = (psi.data_ptr(), state.psi_hat._version) if self.fused else None

    @staticmethod
    def reduce_diag(d: np.ndarray) -> tuple[float, float, float, bool]:
        d = d.reshape(-1, nat.DIAG_SLOTS, nat.DIAG_VALS)
        return (d[..., 0].max(axis=1), d[..., 1].max(axis=1), d[..., 2].max(axis=1),
                d[..., 3].max(axis=1) > 0)

    def _unfused(self, state, params, kx, ky, kz, dptr, st) -> None:
        w = self.worker
        g = self.g
        phys = distfft.inverse(state.psi_hat, w)
        data = phys.dev
        nat.call("pfcs_pfc_cube", nat.ptr(data), data.numel(), 1 if self.real else 0, dptr, st)
        nl_hat = distfft.forward(phys, w)
        nat.call("pfcs_pfc_update", nat.ptr(nl_hat.dev), nat.ptr(state.psi_hat.dev), g.cx, g.ny, g.nz,
                 kx, ky, kz, float(state.symbols.eps), float(params.dt), dptr, st)


def slab_kvectors(grid: GridSpec, sym: SymbolTable, g: _Geometry, device):
    """Device wavenumber vectors (kx, ky, kz) of this rank's spectral slab in
    the kernels' (x', y', z') view (2D grids run as (nx, 1, ny)).

    The C2C slab takes kx from the symbol table (already restricted to the
    X slab, grid.py:178-181); the half-spectrum slab takes rows
    xoff..xoff+cx of the first nx/2+1 entries of the same fftfreq vector
    (their squares — all the PFC multipliers use — are the full grid's)."""
    if g.real:
        kx_np = wavenumbers(grid, 0)[: g.nxm][g.xoff: g.xoff + g.cx]
    else:
        kx_np = sym.kvec[0]
        if kx_np.shape[0] == g.nx and g.cx != g.nx:  # full-grid table: take this rank's rows
            kx_np = kx_np[g.xoff: g.xoff + g.cx]
        if kx_np.shape[0] != g.cx:
            raise ValueError(f"symbol table has {kx_np.shape[0]} x modes, slab has {g.cx}")
    ky_np, kz_np = sym.kvec[1], sym.kvec[2]
    if grid.is_2d:
        ky_np, kz_np = kz_np, ky_np
    return tuple(torch.as_tensor(np.ascontiguousarray(v), dtype=torch.float64, device=device)
                 for v in (kx_np, ky_np, kz_np))


def _is_pencil(field: DistField) -> bool:
    return not isinstance(field.layout, Layout)


def _engine(state: PfcState):
    eng = state._engine
    if eng is None or eng.real != state.psi_hat.half or eng.worker is not state.worker \
            or eng.device != state.psi_hat.dev.device:
        if _is_pencil(state.psi_hat):
            from .pencil import PencilStepEngine

            eng = PencilStepEngine(state)
        else:
            eng = _StepEngine(state)
        state._engine = eng
    return eng


def _spectral_geometry(state: PfcState):
    """(cx, cy, nz, owns_zero_mode, (kx, ky, kz)) of this rank's spectral
    block in the kernels' view, for slabs and pencils alike."""
    w = state.worker
    dev = state.psi_hat.dev.device
    if _is_pencil(state.psi_hat):
        from .pencil import PencilGeometry, pencil_kvectors

        g = PencilGeometry(state.grid, state.psi_hat.layout.grid, w.rank, state.psi_hat.half)
        return g.cx, g.cy2, g.nz, (g.xoff == 0 and g.yoff2 == 0), pencil_kvectors(state.grid, g, dev)
    g = _Geometry(state.grid, w.size, w.rank, state.psi_hat.half)
    return g.cx, g.ny, g.nz, g.xoff == 0, slab_kvectors(state.grid, state.symbols, g, dev)


def _finish(state: PfcState, params: PfcParams, d: np.ndarray, first_index: int,
            realness: list | None = None) -> None:
    m_re, m_im, m_abs, bad = _StepEngine.reduce_diag(d)
    for s in range(len(m_re)):
        if state.psi_hat.dev.numel():
            state.last_max_imag_ratio = float(m_im[s] / m_re[s]) if m_re[s] > 0 else 0.0
        if realness is not None:
            realness.append(state.last_max_imag_ratio)
        if bad[s]:
            state.step_index = first_index + s
            raise DivergenceError(first_index + s, float(m_abs[s]))
    state.step_index = first_index + len(m_re)
    for _ in range(len(m_re)):
        state.sim_time += params.dt


def pfc_step(state: PfcState, params: PfcParams) -> PfcState:
    """Advance one semi-implicit step in place (pfc.py:96-128).  Reads the
    step's diagnostics back (one small device->host copy) so a non-finite
    field raises DivergenceError at this step, as in the reference."""
    eng = _engine(state)
    eng.diag.zero_()
    eng.launch(state, params, eng.diag)
    _finish(state, params, eng.diag.cpu().numpy(), state.step_index)
    return state


def pfc_run(state: PfcState, params: PfcParams, n_steps: int, realness: list | None = None) -> PfcState:
    """``n_steps`` steps enqueued back to back without host round trips (the
    hot loop): per-step diagnostics land in a device array that is read once
    at the end (``realness`` collects each step's max|Im psi|/max|Re psi|).
    Divergence is still reported with the index of the first
    non-finite step (the state has then advanced past it)."""
    n_steps = int(n_steps)
    if n_steps <= 0:
        return state
    eng = _engine(state)
    per = nat.DIAG_SLOTS * nat.DIAG_VALS
    diag = torch.zeros(n_steps * per, dtype=torch.float64, device=eng.device)
    first = state.step_index
    s = 0
    graph = _graph_for(eng, state, params, n_steps)
    if graph is not None:
        # single-rank fused path: replay a captured block of K steps (CUDA
        # graph) — small grids are launch-bound (the 2D 256^2 step is ~us)
        eng.launch(state, params, diag[:per])  # prepares the send buffer
        s = 1
        g, K, dblock = graph
        while n_steps - s >= K:
            g.replay()
            diag[s * per:(s + K) * per].copy_(dblock)
            s += K
        state.psi_hat._version += 1  # replays updated psi_hat in place
        eng.prepared_for = (state.psi_hat.dev.data_ptr(), state.psi_hat._version)
    while s < n_steps:
        eng.launch(state, params, diag[s * per:(s + 1) * per])
        s += 1
    _finish(state, params, diag.cpu().numpy(), first, realness)
    return state


GRAPH_BLOCK = 16
GRAPH_MAX_POINTS = 1 << 22  # graphs only where launch overhead matters


def _graph_for(eng, state: PfcState, params: PfcParams, n_steps: int):
    """Captured K-step block for the single-rank fused engine, or None."""
    if not isinstance(eng, _StepEngine) or eng.G != 1 or not eng.fused:
        return None
    if n_steps <= GRAPH_BLOCK or state.grid.num_points > GRAPH_MAX_POINTS:
        return None
    psi = state.psi_hat.dev
    key = (psi.data_ptr(), float(params.dt), float(state.symbols.eps), id(state.symbols))
    cached = getattr(eng, "_graph", None)
    if cached is not None and cached[0] == key:
        return cached[1]
    per = nat.DIAG_SLOTS * nat.DIAG_VALS
    K = GRAPH_BLOCK
    dblock = torch.zeros(K * per, dtype=torch.float64, device=eng.device)
    # warm the kernels/occupancy caches outside capture, then capture K steps
    # that each start from a prepared send buffer
    eng.prepared_for = None
    side = torch.cuda.Stream(device=eng.device)
    side.wait_stream(torch.cuda.current_stream())
    saved = psi.clone()
    with torch.cuda.stream(side):
        eng.launch(state, params, dblock[:per])  # warm-up step, prepares next
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        dblock.zero_()
        for s in range(K):
            eng.prepared_for = (psi.data_ptr(), state.psi_hat._version)
            eng.launch(state, params, dblock[s * per:(s + 1) * per])
    torch.cuda.current_stream().wait_stream(side)
    psi.copy_(saved)  # capture did not run; undo the warm-up step
    state.psi_hat._version += 1
    eng.prepared_for = None
    eng._graph = (key, (g, K, dblock))
    return eng._graph[1]


def _reduce_sum(worker, value: float) -> float:
    """Rank-ordered scalar sum, identical on every rank (pfc.py:131-137)."""
    total = 0.0
    for p in worker.all_to_all([float(value)] * worker.size):
        total += p
    return total


def _reduce_max(worker, value: float) -> float:
    return max(worker.all_to_all([float(value)] * worker.size))


def _real_part(t: torch.Tensor) -> tuple[torch.Tensor, int]:
    """(float64 view, stride) of the real part of a slab."""
    if t.is_complex():
        return torch.view_as_real(t.reshape(-1)).reshape(-1), 2
    return t.reshape(-1), 1


def free_energy(state: PfcState, params: PfcParams) -> float:
    """sum dV [psi (eps+L) psi / 2 + psi^4 / 4], rank-ordered (pfc.py:144-162)."""
    w = state.worker
    dev = state.psi_hat.dev.device
    st = nat.stream_ptr()
    psi = distfft.inverse(state.psi_hat, w).dev
    cx, cy, nz, _, (kx, ky, kz) = _spectral_geometry(state)
    op_hat = torch.empty_like(state.psi_hat.dev)
    nat.call("pfcs_apply_op", nat.ptr(state.psi_hat.dev), nat.ptr(op_hat), cx, cy, nz,
             nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), float(state.symbols.eps), st)
    op_field = DistField(state.grid, state.psi_hat.layout, Space.SPECTRAL, op_hat,
                         half=state.psi_hat.half, device=dev)
    op_psi = distfft.inverse(op_field, w).dev
    a, sa = _real_part(psi)
    b, sb = _real_part(op_psi)
    n = psi.numel()
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    scratch = torch.empty(max(1, nat.load().pfcs_energy_scratch_bytes(n) // 8), dtype=torch.float64,
                          device=dev)
    nat.call("pfcs_energy_sum", nat.ptr(a), sa, nat.ptr(b), sb, n, nat.ptr(out), nat.ptr(scratch), st)
    local = float(out.item()) * state.grid.cell_volume
    return _reduce_sum(w, local)


def mean_and_max(state: PfcState) -> tuple[float, float]:
    """(mean psi from the zero mode, max |psi|) — collective (pfc.py:165-182)."""
    w = state.worker
    f = state.psi_hat
    owns_zero = _spectral_geometry(state)[3]
    local_zero = 0.0
    if owns_zero and f.dev.numel():
        local_zero = float(f.dev.reshape(-1)[0].real.item())
    zero_mode = _reduce_sum(w, local_zero)
    psi = distfft.inverse(f, w).dev
    a, sa = _real_part(psi)
    out = torch.zeros(1, dtype=torch.float64, device=psi.device)
    nat.call("pfcs_absmax", nat.ptr(a), sa, psi.numel(), nat.ptr(out), nat.stream_ptr())
    local_max = float(out.item()) if psi.numel() else 0.0
    return zero_mode / state.grid.num_points, _reduce_max(w, local_max)


# ----------------------------------------------------- initial conditions ----
# Setup only (not on the hot path); same generators and arithmetic as
# pfc.py:185-310 so runs start from bit-identical fields.

def default_domain_length(n: tuple[int, int, int], points_per_period: int = 8) -> tuple:
    """Lengths commensurate with the lattice wavenumbers (pfc.py:185-201)."""
    nx, ny, nz = n
    if nz == 1:
        return (max(1, nx // points_per_period) * (2.0 * math.pi / TRIANGULAR_Q),
                max(1, ny // (2 * points_per_period)) * (4.0 * math.pi),
                1.0)
    period = 2.0 * math.pi / FCC_Q1
    return tuple(max(1, m // points_per_period) * period for m in n)


def _check_commensurate(grid: GridSpec, q: float, axis: int, mode: str) -> None:
    ratio = grid.length[axis] * q / (2.0 * math.pi)
    if abs(ratio - round(ratio)) > 1e-9:
        msg = (f"domain length {grid.length[axis]} along axis {axis} is not "
               f"commensurate with lattice wavenumber {q} (L*q/2pi = {ratio})")
        if mode == "error":
            raise IncommensurateDomainError(msg)
        warnings.warn(msg, stacklevel=3)


def _axes(grid: GridSpec):
    xs = [np.arange(m) * (grid.length[a] / m) for a, m in enumerate(grid.n)]
    return xs[0][:, None, None], xs[1][None, :, None], xs[2][None, None, :]


def _triangular(x, y, amp: float):
    q = TRIANGULAR_Q
    return amp * (np.cos(q * x) * np.cos(q * y / math.sqrt(3.0))
                  - 0.5 * np.cos(2.0 * q * y / math.sqrt(3.0)))


def _fcc(x, y, z, a1: float, a2: float):
    q = FCC_Q1
    return (8.0 * a1 * np.cos(q * x) * np.cos(q * y) * np.cos(q * z)
            + 2.0 * a2 * (np.cos(2.0 * q * x) + np.cos(2.0 * q * y) + np.cos(2.0 * q * z)))


def initial_field(kind: str, grid: GridSpec, *, psi_bar: float = -0.3, seed: int = 0,
                  noise_amplitude: float = 0.01, amplitude: float = 0.1,
                  amplitude2: float | None = None, n_seeds: int = 5,
                  seed_radius: float | None = None, on_incommensurate: str = "warn") -> np.ndarray:
    """Full-grid initial density, deterministic per seed (pfc.py:237-298)."""
    kind = kind.lower()
    if kind not in INIT_KINDS:
        raise ValueError(f"unknown init kind {kind!r}; expected one of {INIT_KINDS}")
    x, y, z = _axes(grid)
    psi = np.full(grid.shape, psi_bar, dtype=np.float64)
    a2 = amplitude if amplitude2 is None else amplitude2
    if kind == "constant_plus_noise":
        gen = np.random.default_rng(seed)
        return psi + gen.uniform(-noise_amplitude, noise_amplitude, grid.shape)
    if kind == "single_mode_triangular_2d":
        if not grid.is_2d:
            raise ValueError("single_mode_triangular_2d requires nz == 1")
        _check_commensurate(grid, TRIANGULAR_Q, 0, on_incommensurate)
        _check_commensurate(grid, TRIANGULAR_Q / math.sqrt(3.0), 1, on_incommensurate)
        return psi + _triangular(x, y, amplitude)
    if kind == "two_mode_fcc_3d":
        if grid.is_2d:
            raise ValueError("two_mode_fcc_3d requires nz > 1")
        for axis in range(3):
            _check_commensurate(grid, FCC_Q1, axis, on_incommensurate)
        return psi + _fcc(x, y, z, amplitude, a2)
    # seeded_crystallites
    gen = np.random.default_rng(seed)
    radius = seed_radius if seed_radius is not None else 0.15 * min(
        grid.length[:2] if grid.is_2d else grid.length)
    for _ in range(n_seeds):
        c = [gen.uniform(0, grid.length[i]) for i in range(3)]
        if grid.is_2d:
            c[2] = 0.0
            th = gen.uniform(0, 2 * math.pi)
            cs, sn = math.cos(th), math.sin(th)
            dx, dy = x - c[0], y - c[1]
            prof = _triangular(cs * dx - sn * dy, sn * dx + cs * dy, amplitude)
            r2 = dx**2 + dy**2
        else:
            rot = np.linalg.qr(gen.standard_normal((3, 3)))[0]
            dx, dy, dz = x - c[0], y - c[1], z - c[2]
            xr = rot[0, 0] * dx + rot[0, 1] * dy + rot[0, 2] * dz
            yr = rot[1, 0] * dx + rot[1, 1] * dy + rot[1, 2] * dz
            zr = rot[2, 0] * dx + rot[2, 1] * dy + rot[2, 2] * dz
            prof = _fcc(xr, yr, zr, amplitude, a2)
            r2 = dx**2 + dy**2 + dz**2
        env = 0.5 * (1.0 - np.tanh((np.sqrt(r2) - radius) / max(radius * 0.2, 1e-12)))
        psi = psi + env * np.broadcast_to(prof, grid.shape)
    return psi


NOISE_CHUNK_BYTES = 1 << 27  # x-chunk of the streamed noise draw (128 MiB)


def initial_field_slab(kind: str, grid: GridSpec, axis: int, start: int, stop: int, *,
                       psi_bar: float = -0.3, seed: int = 0, noise_amplitude: float = 0.01,
                       amplitude: float = 0.1, amplitude2: float | None = None, n_seeds: int = 5,
                       seed_radius: float | None = None, on_incommensurate: str = "warn") -> np.ndarray:
    """``initial_field(...)[slab]`` for planes [start, stop) of ``axis``,
    bit-identical, without materialising the full grid:
    the per-axis coordinate / cosine vectors are built over the whole axis
    exactly as in ``initial_field`` and then sliced, the pointwise formulas
    are elementwise, and the noise generator is streamed in x-chunks of the
    full grid (the slowest axis, so the draw sequence is the one-shot
    sequence) keeping only the slab's columns.  Memory: the slab plus one
    ~128 MiB chunk, so a 2048^3 run never holds the 64 GiB field on a rank."""
    kind = kind.lower()
    if kind not in INIT_KINDS:
        raise ValueError(f"unknown init kind {kind!r}; expected one of {INIT_KINDS}")
    nx, ny, nz = grid.shape
    sel = [slice(None)] * 3
    sel[axis] = slice(start, stop)
    sel = tuple(sel)
    shape = list(grid.shape)
    shape[axis] = stop - start
    psi = np.full(tuple(shape), psi_bar, dtype=np.float64)
    if kind == "constant_plus_noise":
        gen = np.random.default_rng(seed)
        if axis == 0:
            # draws before the slab's x rows are consumed and discarded in chunks
            row = ny * nz
            x0 = 0
            xc = max(1, NOISE_CHUNK_BYTES // (8 * row))
            while x0 < start:
                m = min(xc, start - x0)
                gen.uniform(-noise_amplitude, noise_amplitude, (m, ny, nz))
                x0 += m
            return psi + gen.uniform(-noise_amplitude, noise_amplitude, tuple(shape))
        noise = np.empty(tuple(shape), dtype=np.float64)
        xc = max(1, NOISE_CHUNK_BYTES // (8 * ny * nz))
        for x0 in range(0, nx, xc):
            x1 = min(nx, x0 + xc)
            blk = gen.uniform(-noise_amplitude, noise_amplitude, (x1 - x0, ny, nz))
            noise[x0:x1] = blk[(slice(None),) + sel[1:]]
        return psi + noise
    x, y, z = _axes(grid)
    cut = lambda v, a: v[sel] if a == axis else v  # noqa: E731
    x, y, z = cut(x, 0), cut(y, 1), cut(z, 2)
    a2 = amplitude if amplitude2 is None else amplitude2
    if kind == "single_mode_triangular_2d":
        if not grid.is_2d:
            raise ValueError("single_mode_triangular_2d requires nz == 1")
        _check_commensurate(grid, TRIANGULAR_Q, 0, on_incommensurate)
        _check_commensurate(grid, TRIANGULAR_Q / math.sqrt(3.0), 1, on_incommensurate)
        return psi + _triangular(x, y, amplitude)
    if kind == "two_mode_fcc_3d":
        if grid.is_2d:
            raise ValueError("two_mode_fcc_3d requires nz > 1")
        for ax in range(3):
            _check_commensurate(grid, FCC_Q1, ax, on_incommensurate)
        return psi + _fcc(x, y, z, amplitude, a2)
    # seeded_crystallites: scalar draws per seed, elementwise envelopes
    gen = np.random.default_rng(seed)
    radius = seed_radius if seed_radius is not None else 0.15 * min(
        grid.length[:2] if grid.is_2d else grid.length)
    for _ in range(n_seeds):
        c = [gen.uniform(0, grid.length[i]) for i in range(3)]
        if grid.is_2d:
            c[2] = 0.0
            th = gen.uniform(0, 2 * math.pi)
            cs, sn = math.cos(th), math.sin(th)
            dx, dy = x - c[0], y - c[1]
            prof = _triangular(cs * dx - sn * dy, sn * dx + cs * dy, amplitude)
            r2 = dx**2 + dy**2
        else:
            rot = np.linalg.qr(gen.standard_normal((3, 3)))[0]
            dx, dy, dz = x - c[0], y - c[1], z - c[2]
            xr = rot[0, 0] * dx + rot[0, 1] * dy + rot[0, 2] * dz
            yr = rot[1, 0] * dx + rot[1, 1] * dy + rot[1, 2] * dz
            zr = rot[2, 0] * dx + rot[2, 1] * dy + rot[2, 2] * dz
            prof = _fcc(xr, yr, zr, amplitude, a2)
            r2 = dx**2 + dy**2 + dz**2
        env = 0.5 * (1.0 - np.tanh((np.sqrt(r2) - radius) / max(radius * 0.2, 1e-12)))
        psi = psi + env * np.broadcast_to(prof, tuple(shape))
    return psi


def init_condition(kind: str, grid: GridSpec, worker, *, real: bool = False, **kwargs) -> DistField:
    """Initial density in the physical layout (pfc.py:301-310).  Each rank
    builds only its own slab (``initial_field_slab``; bit-identical to the
    reference's scatter of the replicated full field).  ``real=True`` keeps
    the slab float64 (R2C/C2R path)."""
    layout = distfft.physical_layout(grid)
    lay = distfft.layout_for(grid, layout, worker.size)
    r = worker.rank
    part = initial_field_slab(kind, grid, lay.axis, lay.offsets[r], lay.offsets[r] + lay.counts[r], **kwargs)
    dtype = np.float64 if real else np.complex128
    return DistField(grid, layout, Space.PHYSICAL, np.ascontiguousarray(part, dtype=dtype),
                     device=distfft._device_of(worker))
