"""Hydrodynamic PFC, field-per-GPU (drop-in for hydro.py).

Reference: /root/reference/pkg/src/pfcspectral/hydro.py:1-165 — density psi
coupled to a coarse-grained velocity (v1, v2, v3):

    psi_hat <- (psi_hat + dt*(lap*F[psi^3] - F[v . grad psi])) / (1 - dt*lin)
    v_hat_i <- (v_hat_i - (dt/rho)*cg*F[psi * d_i(mu)]) / (1 - (dt/rho)*gamma*lap)

Parallel strategy (paper strategy 2, hydro.py:129-156): one field per GPU —
rank 0 owns psi, ranks 1..3 own v1..v3 — with the physical psi broadcast
from rank 0 (tag 2) and the physical velocities returned (tags 4, 5, 6)
once per step.  Fields are full-grid complex128 CUDA tensors; transforms are
the libpfcs line kernels (serial 3D FFT, one HBM pass per axis) and the
pointwise operators are libpfcs kernels in numpy's evaluation order
(csrc/pfcs_hydro.cu).  numpy inputs are accepted (and numpy returned) for
drop-in use; CUDA tensors stay on the device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field as dataclass_field

import numpy as np
import torch

from . import _native as nat
from .grid import GridSpec, SymbolTable
from .pfc import DivergenceError, PfcParams

__all__ = [
    "HydroParams",
    "HydroFields",
    "TAG_PSI",
    "V_TAGS",
    "hydro_psi_step",
    "hydro_velocity_step",
    "serial_hydro_step",
    "parallel_hydro_step",
    "free_energy_full",
]

TAG_PSI = 2
V_TAGS = (4, 5, 6)


@dataclass
class HydroParams:
    pfc: PfcParams = dataclass_field(default_factory=PfcParams)
    rho: float = 1.0
    gamma: float = 1.0
    a0: float = 2.0 * math.pi

    def __post_init__(self):
        if not (self.rho > 0 and math.isfinite(self.rho)):
            raise ValueError(f"rho must be positive, got {self.rho}")
        if not (self.gamma >= 0 and math.isfinite(self.gamma)):
            raise ValueError(f"gamma must be >= 0, got {self.gamma}")
        if not (self.a0 > 0 and math.isfinite(self.a0)):
            raise ValueError(f"a0 must be positive, got {self.a0}")


@dataclass
class HydroFields:
    """Full-grid state of the serial mode (hydro.py:60-69)."""

    psi_hat: object
    psi: object
    v_hat: list
    v: list
    step_index: int = 0
    sim_time: float = 0.0


# ------------------------------------------------------------------ helpers --

def _dev(x) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            nat.load()
            x = x.cuda()
        return x.to(torch.complex128).contiguous()
    nat.load()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    return torch.from_numpy(arr).to(torch.device("cuda", torch.cuda.current_device()))


def _out(t: torch.Tensor, host: bool):
    return t.cpu().numpy() if host else t


PRO_CUBE, PRO_CMUL, PRO_DERIV = 1, 2, 3  # fused prologues (include/pfcs.h pfcs_fft_axis_c2c_pro)


def _fft(t: torch.Tensor, forward: bool, pro: int = 0, aux=None, aux_axis: int = 0) -> torch.Tensor:
    """Full-grid 3D transform, one libpfcs pass per axis (orders as
    fftcore.fft_nd: forward 0,1,2; inverse 2,1,0).  ``pro`` fuses a pointwise
    product into the first pass: F(t^3), F(aux * t), F^-1(i d_axis t)."""
    out = torch.empty_like(t)
    n0, n1, n2 = t.shape
    st = nat.stream_ptr()
    order = (0, 1, 2) if forward else (2, 1, 0)
    src = t
    for k, ax in enumerate(order):
        if k == 0 and pro:
            nat.call("pfcs_fft_axis_c2c_pro", nat.ptr(src), nat.ptr(out), n0, n1, n2, ax, 1 if forward else 0,
                     pro, nat.ptr(aux) if aux is not None else None, aux_axis, st)
        else:
            nat.call("pfcs_fft_axis_c2c", nat.ptr(src), nat.ptr(out), n0, n1, n2, ax, 1 if forward else 0, st)
        src = out
    return out


def _fft_cube(ps: torch.Tensor) -> torch.Tensor:
    """F(psi**3) with the cube fused into the first (x) pass."""
    return _fft(ps, True, PRO_CUBE)


def _fft_cmul(a: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    """F(a * g) with the product fused into the first (x) pass."""
    return _fft(g, True, PRO_CMUL, a)


def _ifft_deriv(x_hat: torch.Tensor, axis: int, sym) -> torch.Tensor:
    """F^-1(i k_axis x_hat) with the multiplier fused into the first (z) pass."""
    return _fft(x_hat, False, PRO_DERIV, _vectors(sym, x_hat.device)[3 + axis], axis)


def _cube(t: torch.Tensor) -> torch.Tensor:
    c = t.clone()
    nat.call("pfcs_pfc_cube", nat.ptr(c), c.numel(), 0, None, nat.stream_ptr())
    return c


def _vectors(sym: SymbolTable, device):
    return sym.device_vectors(device)


def _deriv_axis(d_axis, sym: SymbolTable):
    """Which i*k_axis multiplier the caller passed (sym.d1/d2/d3 or an int)."""
    if isinstance(d_axis, (int, np.integer)):
        return int(d_axis)
    cache = sym.__dict__.get("_cache", {})
    for ax in range(3):
        if cache.get(f"d{ax + 1}") is d_axis:
            return ax
    return None


def _mul_deriv(x: torch.Tensor, axis, d_axis, sym) -> torch.Tensor:
    out = torch.empty_like(x)
    st = nat.stream_ptr()
    if axis is not None:
        dvec = _vectors(sym, x.device)[3 + axis]
        n0, n1, n2 = x.shape
        nat.call("pfcs_mul_deriv", nat.ptr(x), nat.ptr(out), n0, n1, n2, nat.ptr(dvec), axis, st)
    else:  # an arbitrary multiplier array
        d = _dev(d_axis)
        nat.call("pfcs_cmul", nat.ptr(d), nat.ptr(x), nat.ptr(out), x.numel(), st)
    return out


class _Diag:
    def __init__(self, device):
        self.t = torch.zeros(nat.DIAG_SLOTS * nat.DIAG_VALS, dtype=torch.float64, device=device)

    def bad(self) -> bool:
        return bool(self.t.view(nat.DIAG_SLOTS, nat.DIAG_VALS)[:, 3].max().item() > 0)


def _raise_divergence(step_index: int, a: torch.Tensor):
    m = torch.abs(a)
    m = m[~torch.isnan(m)]
    raise DivergenceError(step_index, float(m.max().item()) if m.numel() else float("nan"))


# -------------------------------------------------------------- the steps ----

def hydro_psi_step(psi_hat, psi, v1, v2, v3, sym: SymbolTable, params: HydroParams,
                   step_index: int = 0):
    """Advect-and-relax update of the density (hydro.py:77-90); returns
    (psi_hat, psi) as new arrays."""
    host = isinstance(psi_hat, np.ndarray)
    ph, ps = _dev(psi_hat), _dev(psi)
    vs = [_dev(v) for v in (v1, v2, v3)]
    dev = ph.device
    kx, ky, kz = _vectors(sym, dev)[:3]
    n0, n1, n2 = ph.shape
    st = nat.stream_ptr()
    xs = [_ifft_deriv(ph, ax, sym) for ax in range(3)]
    adv = torch.empty_like(ph)
    nat.call("pfcs_hydro_advect", nat.ptr(vs[0]), nat.ptr(xs[0]), nat.ptr(vs[1]), nat.ptr(xs[1]),
             nat.ptr(vs[2]), nat.ptr(xs[2]), nat.ptr(adv), adv.numel(), st)
    del xs
    nl_hat = _fft_cube(ps)
    adv_hat = _fft(adv, True)
    new = torch.empty_like(ph)
    diag = _Diag(dev)
    nat.call("pfcs_hydro_psi_update_to", nat.ptr(ph), nat.ptr(new), nat.ptr(nl_hat), nat.ptr(adv_hat), n0, n1, n2,
             nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), float(sym.eps), float(params.pfc.dt),
             nat.ptr(diag.t), st)
    if diag.bad():
        _raise_divergence(step_index, new)
    new_psi = _fft(new, False)
    return _out(new, host), _out(new_psi, host)


def _mu_hat(ps: torch.Tensor, sym: SymbolTable) -> torch.Tensor:
    """mu_hat = F[psi^3] + op F[psi] (hydro.py:96-97)."""
    kx, ky, kz = _vectors(sym, ps.device)[:3]
    n0, n1, n2 = ps.shape
    nl_hat = _fft_cube(ps)
    f_hat = _fft(ps, True)
    mu_hat = torch.empty_like(ps)
    nat.call("pfcs_hydro_mu", nat.ptr(nl_hat), nat.ptr(f_hat), nat.ptr(mu_hat), n0, n1, n2,
             nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), float(sym.eps), nat.stream_ptr())
    return mu_hat


def hydro_velocity_step(v_hat, psi, d_axis, sym: SymbolTable, params: HydroParams,
                        step_index: int = 0, *, mu_hat=None):
    """Viscous decay plus Gaussian-smoothed thermodynamic force on one
    velocity component (hydro.py:93-107); ``d_axis`` is sym.d1/d2/d3 (or
    the axis index).  Returns (v_hat, v) as new arrays."""
    host = isinstance(v_hat, np.ndarray)
    vh, ps = _dev(v_hat), _dev(psi)
    dev = vh.device
    kx, ky, kz = _vectors(sym, dev)[:3]
    n0, n1, n2 = vh.shape
    st = nat.stream_ptr()
    axis = _deriv_axis(d_axis, sym)
    if mu_hat is None:  # shared by the three components in serial mode
        mu_hat = _mu_hat(ps, sym)
    if axis is not None:
        g = _ifft_deriv(mu_hat, axis, sym)
    else:
        g = _fft(_mul_deriv(mu_hat, axis, d_axis, sym), False)
    force = _fft_cmul(ps, g)  # F(psi * g), product fused into the first pass
    dt, rho = float(params.pfc.dt), float(params.rho)
    new = torch.empty_like(vh)
    diag = _Diag(dev)
    nat.call("pfcs_hydro_vel_update_to", nat.ptr(vh), nat.ptr(new), nat.ptr(force), n0, n1, n2, nat.ptr(kx), nat.ptr(ky),
             nat.ptr(kz), dt / rho, (dt / rho) * float(params.gamma), -0.5 * float(sym.a0) ** 2,
             nat.ptr(diag.t), st)
    if diag.bad():
        _raise_divergence(step_index, new)
    v = _fft(new, False)
    return _out(new, host), _out(v, host)


def serial_hydro_step(fields: HydroFields, sym: SymbolTable, params: HydroParams) -> HydroFields:
    """The four-role dataflow on one worker (hydro.py:110-126): density
    first with the previous velocities, then v1..v3 with the fresh density."""
    fields.psi_hat, fields.psi = hydro_psi_step(fields.psi_hat, fields.psi, *fields.v, sym, params,
                                                step_index=fields.step_index)
    ps = _dev(fields.psi)
    mu_hat = _mu_hat(ps, sym)  # the three components share it
    for i in range(3):
        fields.v_hat[i], fields.v[i] = hydro_velocity_step(fields.v_hat[i], ps, i, sym, params,
                                                           step_index=fields.step_index, mu_hat=mu_hat)
    fields.step_index += 1
    fields.sim_time += params.pfc.dt
    return fields


def parallel_hydro_step(worker, role_state: dict, sym: SymbolTable, params: HydroParams) -> dict:
    """One step of the four-GPU dataflow (hydro.py:129-156): rank 0 owns
    psi, rank i owns v_i; psi goes out on tag 2, v_i comes back on tag 3+i.
    Device tensors travel as device messages (NCCL p2p between processes,
    device copies between threads); host arrays as host objects."""
    rank = worker.rank
    device_msgs = isinstance(role_state.get("psi"), torch.Tensor)
    if rank == 0:
        psi_hat, psi = hydro_psi_step(role_state["psi_hat"], role_state["psi"], *role_state["v"], sym,
                                      params, step_index=role_state["step_index"])
        role_state["psi_hat"], role_state["psi"] = psi_hat, psi
        for dst in (1, 2, 3):
            if device_msgs:
                worker.send_tensor(dst, TAG_PSI, psi)
            else:
                worker.send(dst, TAG_PSI, psi)
        if device_msgs:
            role_state["v"] = [worker.recv_tensor(i + 1, V_TAGS[i], torch.empty_like(psi))
                               for i in range(3)]
        else:
            role_state["v"] = [worker.receive(i + 1, V_TAGS[i]) for i in range(3)]
    else:
        i = rank - 1
        if device_msgs:
            psi = worker.recv_tensor(0, TAG_PSI, torch.empty_like(role_state["psi"]))
        else:
            psi = worker.receive(0, TAG_PSI)
        role_state["psi"] = psi
        v_hat, v = hydro_velocity_step(role_state["v_hat"], psi, i, sym, params,
                                       step_index=role_state["step_index"])
        role_state["v_hat"], role_state["v_own"] = v_hat, v
        if device_msgs:
            worker.send_tensor(0, V_TAGS[i], v)
        else:
            worker.send(0, V_TAGS[i], v)
    role_state["step_index"] += 1
    return role_state


def free_energy_full(psi, sym: SymbolTable, grid: GridSpec) -> float:
    """Free energy of a full-grid density (hydro.py:159-165)."""
    ps = _dev(psi)
    dev = ps.device
    kx, ky, kz = _vectors(sym, dev)[:3]
    n0, n1, n2 = ps.shape
    st = nat.stream_ptr()
    f = _fft(ps, True)
    op_f = torch.empty_like(f)
    nat.call("pfcs_apply_op", nat.ptr(f), nat.ptr(op_f), n0, n1, n2, nat.ptr(kx), nat.ptr(ky), nat.ptr(kz),
             float(sym.eps), st)
    op_psi = _fft(op_f, False)
    a = torch.view_as_real(ps.reshape(-1)).reshape(-1)
    b = torch.view_as_real(op_psi.reshape(-1)).reshape(-1)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    n = ps.numel()
    scratch = torch.empty(max(1, nat.load().pfcs_energy_scratch_bytes(n) // 8), dtype=torch.float64,
                          device=dev)
    nat.call("pfcs_energy_sum", nat.ptr(a), 2, nat.ptr(b), 2, n, nat.ptr(out), nat.ptr(scratch), st)
    return float(out.item()) * grid.cell_volume
