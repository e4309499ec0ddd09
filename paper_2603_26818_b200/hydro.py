"""Hydrodynamic PFC, field-per-GPU (drop-in for hydro.py).

Reference: /root/reference/pkg/src/pfcspectral/hydro.py:1-165 — density psi
coupled to a coarse-grained velocity (v1, v2, v3):

    psi_hat <- (psi_hat + dt*(lap*F[psi^3] - F[v . grad psi])) / (1 - dt*lin)
    v_hat_i <- (v_hat_i - (dt/rho)*cg*F[psi * d_i(mu)]) / (1 - (dt/rho)*gamma*lap)

Parallel strategy (paper strategy 2, hydro.py:129-156): one field per GPU —
rank 0 owns psi, ranks 1..3 own v1..v3 — with the physical psi broadcast
from rank 0 (tag 2) and the physical velocities returned (tags 4, 5, 6)
once per step.  Complex full-grid fields (the reference's representation)
are transformed C2C by the libpfcs line kernels (one HBM pass per axis) with
the pointwise operators as libpfcs kernels in numpy's evaluation order
(csrc/pfcs_hydro.cu).  Real physical fields (float64 psi, v_i with x-halved
half spectra) take the B200 R2C path at the end of this module: half the
bytes per transform, 8-byte real products (pfcs_real_pointwise), the i k
multipliers fused into the inverse transforms, one divergence read-back per
step; results equal the C2C path to rounding.  numpy inputs are accepted
(and numpy returned) for drop-in use; CUDA tensors stay on the device.
"""

from __future__ import annotations

import math
import os
import weakref
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
    first with the previous velocities, then v1..v3 with the fresh density.
    Real physical fields (float64 psi, v_i; x-halved spectra) take the R2C
    path (module doc)."""
    if _is_real(fields.psi):
        return _serial_hydro_step_r(fields, sym, params)
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
    if device_msgs and not role_state["psi"].is_complex():
        return _parallel_hydro_step_r(worker, role_state, sym, params)
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


# ------------------------------------------------------------ R2C path ------
# Real physical fields (float64) with x-halved spectra: the B200
# representation of the hydro / multiphysics fields (multiphysics.py doc).

RPW_CUBE, RPW_MUL, RPW_ADV3, RPW_CHNL, RPW_ADD3 = 0, 1, 2, 3, 4  # pfcs_real_pointwise kinds
_R2C_PRO = os.environ.get("PFCS_R2C_PRO", "1") != "0"  # fused prologues (A/B switch)
_R2C_UPD = os.environ.get("PFCS_R2C_UPD", "1") != "0"  # updates fused into the next inverse (A/B switch)
# x / y derivatives share one z pass, multiplier in the y pass (A/B timing
# switch: PFCS_R2C_GRAD=0 multiplies in each derivative's own z pass, which
# rounds differently — not a bit-identity switch)
_R2C_GRAD = os.environ.get("PFCS_R2C_GRAD", "1") != "0"
# the force product in one fused x pass (_Real3.prod_grad; A/B, bit-identical)
_R2C_XMUL = os.environ.get("PFCS_R2C_XMUL", "1") != "0"
# the advection dot product in one fused x pass (_Real3.adv_fwd; A/B, bit-identical)
_R2C_XDOT = os.environ.get("PFCS_R2C_XDOT", "1") != "0"
# mu_hat with its operands' forward z passes (pfcs_hydro_mu_z; A/B, bit-identical)
_R2C_MUZ = os.environ.get("PFCS_R2C_MUZ", "1") != "0"
# ... and grad mu's first inverse z passes inside it (pfcs_hydro_mu_zgrad; A/B, bit-identical)
_R2C_MUZG = os.environ.get("PFCS_R2C_MUZG", "1") != "0"
# serial steps carry F(psi^3) from one step's mu to the next step's density
# update (same psi, same spectrum; A/B, bit-identical)
_CARRY_NL = os.environ.get("PFCS_R2C_CARRY", "1") != "0"
# updates take their operands before the forward z pass and run it
# (pfcs_update_zzinv; A/B, bit-identical)
_R2C_ZZ = os.environ.get("PFCS_R2C_ZZ", "1") != "0"


def _is_real(x) -> bool:
    if isinstance(x, torch.Tensor):
        return not x.is_complex()
    return isinstance(x, np.ndarray) and not np.iscomplexobj(x)


def _rdev(x) -> torch.Tensor:
    """float64 CUDA tensor (contiguous) of a real field."""
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.cuda()
        return t.to(torch.float64).contiguous()
    nat.load()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(
        torch.device("cuda", torch.cuda.current_device()))


def _hdev(x) -> torch.Tensor:
    """complex128 CUDA tensor of a half spectrum."""
    return _dev(x)


class _Real3:
    """Full-grid 3D R2C / C2R transforms of an (nx, ny, nz) real field with the
    x axis halved — the layout of the slab pipeline at G = 1 (distfft):
    forward rfft_x, y, z; inverse z, y, irfft_x; the inverse may fuse the
    derivative multiplier i d_axis into its first (z) pass."""

    def __init__(self, shape, sym: SymbolTable, device):
        nx, ny, nz = shape
        if nx < 4 or nx & (nx - 1):
            raise ValueError(f"the R2C multiphysics path needs a power-of-two nx >= 4, got {nx}")
        self.shape = (nx, ny, nz)
        self.nh = nx // 2 + 1
        self.hshape = (self.nh, ny, nz)
        kx, ky, kz, dx, dy, dz = sym.device_vectors(device)
        self.k = (kx[: self.nh].contiguous(), ky, kz)
        self.d = (dx[: self.nh].contiguous(), dy, dz)

    @staticmethod
    def of(shape, sym: SymbolTable, device) -> "_Real3":
        cache = sym.__dict__.setdefault("_real3", {})
        key = (tuple(shape), str(device))
        if key not in cache:
            cache[key] = _Real3(shape, sym, device)
        return cache[key]

    def fwd(self, x: torch.Tensor, kind: int | None = None, aux: torch.Tensor | None = None,
            alpha: float = 0.0, z: bool = True) -> torch.Tensor:
        """F[x], or F[f(x)] with f a pfcs_real_pointwise kind (0 cube, 1 x*aux,
        3 alpha (x^3 - x)) fused into the first (x) pass (PFCS_R2C_PRO=0:
        the product in its own pass, bit-identical).  z=False stops before
        the z pass (for a consumer that fuses it)."""
        nx, ny, nz = self.shape
        out = torch.empty(self.hshape, dtype=torch.complex128, device=x.device)
        st = nat.stream_ptr()
        if kind is not None and not _R2C_PRO:
            x = _rpw(kind, x, *([aux] if aux is not None else []), alpha=alpha)
            kind = None
        if kind is None:
            nat.call("pfcs_rfft_x", nat.ptr(x), nat.ptr(out), nx, ny * nz, st)
        else:
            nat.call("pfcs_rfft_x_pro", nat.ptr(x), nat.ptr(out), nx, ny * nz, kind,
                     nat.ptr(aux) if aux is not None else None, float(alpha), st)
        if ny > 1:
            nat.call("pfcs_fft_axis_c2c", nat.ptr(out), nat.ptr(out), self.nh, ny, nz, 1, 1, st)
        if nz > 1 and z:
            nat.call("pfcs_fft_axis_c2c", nat.ptr(out), nat.ptr(out), self.nh, ny, nz, 2, 1, st)
        return out

    def update_inv(self, kind: int, state: torch.Tensor, aux: torch.Tensor, aux2, c: tuple,
                   flag: "_StepFlag", keep_z: bool = False, pre_z=(False, False)) -> tuple:
        """A spectral update fused with the first (z) pass of the inverse
        transform of its result (pfcs_update_zinv; kind 0 psi, 1 velocity,
        2 composition): returns (new state, F^-1 of it).  PFCS_R2C_UPD=0 runs
        the standalone update kernel and the plain inverse (bit-identical).
        keep_z: also return {"z": the inverse z pass, "y": its y pass} of
        the new state (or None) — the next step's gradient of that state
        starts from them (_grad_zy, adv_fwd), so the serial steps carry them
        over.  pre_z: (aux, aux2)
        arrive before their forward z pass (fwd(..., z=False)); the update
        runs it in registers (pfcs_update_zzinv; PFCS_R2C_ZZ=0: the z passes
        in place first — bit-identical)."""
        nx, ny, nz = self.shape
        nh = self.nh
        kx, ky, kz = self.k
        st = nat.stream_ptr()
        new = torch.empty_like(state)
        pre_z = (bool(pre_z[0]), bool(pre_z[1]) and aux2 is not None)
        fuse_zz = any(pre_z) and _R2C_ZZ and _R2C_UPD and nz > 1
        if any(pre_z) and not fuse_zz and nz > 1:
            for t, pz in ((aux, pre_z[0]), (aux2, pre_z[1])):
                if pz:
                    nat.call("pfcs_fft_axis_c2c", nat.ptr(t), nat.ptr(t), nh, ny, nz, 2, 1, st)
        if not _R2C_UPD:
            name = ("pfcs_hydro_psi_update_to", "pfcs_hydro_vel_update_to", "pfcs_ch_update_to")[kind]
            ops = [nat.ptr(state), nat.ptr(new), nat.ptr(aux)] + ([] if kind == 1 else [nat.ptr(aux2)])
            consts = c[:2] if kind == 0 else c
            nat.call(name, *ops, nh, ny, nz, nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), *(float(v) for v in consts),
                     nat.ptr(flag.t), st)
            return (new, self.inv(new), None) if keep_z else (new, self.inv(new))
        tmp = torch.empty_like(state)
        c3 = tuple(float(v) for v in c) + (0.0,) * (3 - len(c))
        if fuse_zz:
            nat.call("pfcs_update_zzinv", kind, nat.ptr(state), nat.ptr(aux),
                     nat.ptr(aux2) if aux2 is not None else None, nat.ptr(new), nat.ptr(tmp), nh, ny, nz,
                     nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), *c3, int(pre_z[0]) | (2 * int(pre_z[1])),
                     nat.ptr(flag.t), st)
        else:
            nat.call("pfcs_update_zinv", kind, nat.ptr(state), nat.ptr(aux),
                     nat.ptr(aux2) if aux2 is not None else None, nat.ptr(new), nat.ptr(tmp), nh, ny, nz,
                     nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), *c3, nat.ptr(flag.t), st)
        keep = {"z": tmp, "y": None} if keep_z else None
        if ny > 1:
            ybuf = torch.empty_like(tmp) if keep_z else tmp  # (out of place keeps the z pass)
            nat.call("pfcs_fft_axis_c2c", nat.ptr(tmp), nat.ptr(ybuf), nh, ny, nz, 1, 0, st)
            tmp = ybuf
            if keep_z:
                keep["y"] = ybuf  # the C2R below only reads it
        out = torch.empty(self.shape, dtype=torch.float64, device=state.device)
        nat.call("pfcs_irfft_x", nat.ptr(tmp), nat.ptr(out), nx, ny * nz, st)
        return (new, out, keep) if keep_z else (new, out)

    def inv(self, h: torch.Tensor, deriv: int | None = None) -> torch.Tensor:
        """F^-1[h], or F^-1[i d_deriv h] (grad_inv's recipe for that axis)."""
        if deriv is not None:
            return self.grad_inv(h, (deriv,))[0]
        nx, ny, nz = self.shape
        nh = self.nh
        st = nat.stream_ptr()
        tmp = torch.empty_like(h)
        nat.call("pfcs_fft_axis_c2c", nat.ptr(h), nat.ptr(tmp), nh, ny, nz, 2, 0, st)
        if ny > 1:
            nat.call("pfcs_fft_axis_c2c", nat.ptr(tmp), nat.ptr(tmp), nh, ny, nz, 1, 0, st)
        out = torch.empty(self.shape, dtype=torch.float64, device=h.device)
        nat.call("pfcs_irfft_x", nat.ptr(tmp), nat.ptr(out), nx, ny * nz, st)
        return out

    def _grad_zy(self, h: torch.Tensor, axes, outs=None, t0=None, tz=None, x_at_x: bool = False) -> list:
        """The inverse z and y passes of F^-1(i d_a h) for each a in axes
        (x-halved spectra, before the x pass).  k_x and k_y are constant
        along z lines, so the x and y derivatives share ONE plain inverse z
        pass and take their multiplier in the y pass (pfcs_fft_axis_c2c_pro,
        axis 1); the z derivative takes it in its own z pass.  A gradient
        costs two z passes instead of three (2S less HBM traffic).  Every
        caller — the serial steps and each rank of the role maps — forms a
        derivative along a given axis this way, so they stay bit-identical.
        x_at_x: the x derivative's output is the plain y pass of the shared z
        pass — its i d_x (a function of the x mode only) is applied at the
        x stage by the caller (the advection recipe: grad_inv, adv_fwd)."""
        nx, ny, nz = self.shape
        nh = self.nh
        st = nat.stream_ptr()
        share = ny > 1 and _R2C_GRAD
        t0 = t0 if share else None  # the plain inverse z pass of h, when the caller has it
        like = h if h is not None else (t0 if t0 is not None else tz)  # (h is None when t0 / tz cover the axes)
        given, outs = outs, []
        for n_a, a in enumerate(axes):
            tmp = given[n_a] if given is not None else torch.empty_like(like)
            if share and a != 2:
                if t0 is None:
                    t0 = torch.empty_like(h)
                    nat.call("pfcs_fft_axis_c2c", nat.ptr(h), nat.ptr(t0), nh, ny, nz, 2, 0, st)
                if a == 0 and x_at_x:
                    nat.call("pfcs_fft_axis_c2c", nat.ptr(t0), nat.ptr(tmp), nh, ny, nz, 1, 0, st)
                else:
                    nat.call("pfcs_fft_axis_c2c_pro", nat.ptr(t0), nat.ptr(tmp), nh, ny, nz, 1, 0, 3,
                             nat.ptr(self.d[a]), a, st)
            elif tz is not None and share:  # the caller ran the z pass with i d_z (pfcs_hydro_mu_zgrad)
                nat.call("pfcs_fft_axis_c2c", nat.ptr(tz), nat.ptr(tmp), nh, ny, nz, 1, 0, st)
            else:  # i d_a fused into the z pass
                nat.call("pfcs_fft_axis_c2c_pro", nat.ptr(h), nat.ptr(tmp), nh, ny, nz, 2, 0, 3,
                         nat.ptr(self.d[a]), a, st)
                if ny > 1:
                    nat.call("pfcs_fft_axis_c2c", nat.ptr(tmp), nat.ptr(tmp), nh, ny, nz, 1, 0, st)
            outs.append(tmp)
        return outs

    def grad_inv(self, h: torch.Tensor, axes=(0, 1, 2)) -> list:
        """[F^-1(i d_a h) for a in axes] (real fields) in the advection
        recipe (_grad_zy x_at_x: the x derivative's multiplier at the x
        stage, here as pfcs_mul_deriv before the C2R)."""
        nx, ny, nz = self.shape
        nh = self.nh
        st = nat.stream_ptr()
        share = ny > 1 and _R2C_GRAD
        outs = []
        for a, tmp in zip(axes, self._grad_zy(h, axes, x_at_x=True)):
            if a == 0 and share:
                nat.call("pfcs_mul_deriv", nat.ptr(tmp), nat.ptr(tmp), nh, ny, nz, nat.ptr(self.d[0]), 0, st)
            out = torch.empty(self.shape, dtype=torch.float64, device=h.device)
            nat.call("pfcs_irfft_x", nat.ptr(tmp), nat.ptr(out), nx, ny * nz, st)
            outs.append(out)
        return outs

    def adv_fwd(self, x_hat: torch.Tensor, v, t0=None, z: bool = True, y0=None) -> torch.Tensor:
        """F(v . grad x) (hydro.py:83-85): _grad_zy's inverse z / y passes
        into one stacked buffer, ONE fused x pass (pfcs_xdot3_x: the three
        C2R, the dot product with v, the R2C — the physical derivatives and
        the product never reach HBM), the forward y and z passes.
        Bit-identical to fwd(_grad_dot_r(self, x_hat, v)), which runs when
        PFCS_R2C_XDOT=0 or the shape has no fused kernel.  t0 / y0: the
        plain inverse z pass / z and y passes of x_hat if the caller has them
        (update_inv keep_z) — the x derivative takes its i d_x in the x pass
        (_grad_zy x_at_x), so with y0 it needs no pass of its own."""
        nx, ny, nz = self.shape
        if not (_R2C_XDOT and nat.load().pfcs_xdot3_supported(nx, ny * nz)):
            return self.fwd(_grad_dot_r(self, x_hat, v), z=z)
        st = nat.stream_ptr()
        share = ny > 1 and _R2C_GRAD
        if share and y0 is not None:
            specs = [y0] + self._grad_zy(x_hat, (1, 2), t0=t0)
        else:
            specs = self._grad_zy(x_hat, (0, 1, 2), t0=t0, x_at_x=True)
        out = torch.empty(self.hshape, dtype=torch.complex128, device=x_hat.device)
        vs = [_rdev(x) for x in v]
        nat.call("pfcs_xdot3_x", nat.ptr(specs[0]), nat.ptr(specs[1]), nat.ptr(specs[2]), nat.ptr(vs[0]),
                 nat.ptr(vs[1]), nat.ptr(vs[2]), nat.ptr(out), nx, ny * nz,
                 nat.ptr(self.d[0]) if share else None, st)
        if ny > 1:
            nat.call("pfcs_fft_axis_c2c", nat.ptr(out), nat.ptr(out), self.nh, ny, nz, 1, 1, st)
        if nz > 1 and z:
            nat.call("pfcs_fft_axis_c2c", nat.ptr(out), nat.ptr(out), self.nh, ny, nz, 2, 1, st)
        return out

    def prod_grad(self, h: torch.Tensor, aux: torch.Tensor, axes=(0, 1, 2), z: bool = True, zpre=None) -> list:
        """[F(aux * F^-1(i d_a h)) for a in axes] — the hydro force
        F(psi F^-1(i k mu_hat)) (hydro.py:98): the inverse z / y passes of
        _grad_zy, ONE fused x pass (C2R, times aux, R2C: pfcs_xmul_x, the
        physical derivative and the product never reach HBM), the forward y
        and z passes.  Bit-identical to fwd(grad_inv(h)[a], RPW_MUL, aux)
        (PFCS_R2C_XMUL=0 runs that form).  zpre: {"t0", "tz"} — the
        gradient's first inverse z passes when the caller ran them
        (_density_mu_r grad_axes); h may then be None."""
        zpre = zpre or {}
        nx, ny, nz = self.shape
        nh = self.nh
        st = nat.stream_ptr()
        outs = self._grad_zy(h, axes, t0=zpre.get("t0"), tz=zpre.get("tz"))
        if not _R2C_XMUL:
            res = []
            for tmp in outs:
                d = torch.empty(self.shape, dtype=torch.float64, device=tmp.device)
                nat.call("pfcs_irfft_x", nat.ptr(tmp), nat.ptr(d), nx, ny * nz, st)
                res.append(self.fwd(d, RPW_MUL, aux, z=z))
            return res
        for tmp in outs:
            nat.call("pfcs_xmul_x", nat.ptr(tmp), nat.ptr(aux), nx, ny * nz, st)
            if ny > 1:
                nat.call("pfcs_fft_axis_c2c", nat.ptr(tmp), nat.ptr(tmp), nh, ny, nz, 1, 1, st)
            if nz > 1 and z:
                nat.call("pfcs_fft_axis_c2c", nat.ptr(tmp), nat.ptr(tmp), nh, ny, nz, 2, 1, st)
        return outs


def _check_half(R: _Real3, *spectra: torch.Tensor) -> None:
    """The R2C path takes x-halved spectra: a full-grid spectrum next to a
    real field is a representation mix-up, not something to compute on."""
    for h in spectra:
        if tuple(h.shape) != R.hshape or not h.is_complex():
            raise ValueError(f"real physical fields select the R2C path, which needs x-halved complex spectra of "
                             f"shape {R.hshape}; got {tuple(h.shape)} {h.dtype} (pass complex fields for the "
                             f"reference's full-grid C2C representation)")


def _rpw(kind: int, *ops: torch.Tensor, alpha: float = 0.0) -> torch.Tensor:
    out = torch.empty_like(ops[0])
    args = [nat.ptr(o) for o in ops] + [None] * (6 - len(ops))
    nat.call("pfcs_real_pointwise", kind, *args, nat.ptr(out), out.numel(), float(alpha), nat.stream_ptr())
    return out


class _StepFlag:
    """One device diagnostics block shared by a step's spectral updates; the
    non-finite flag is read back once per step (not once per update)."""

    def __init__(self, device):
        self.t = torch.zeros(nat.DIAG_SLOTS * nat.DIAG_VALS, dtype=torch.float64, device=device)

    def check(self, step_index: int, *fields: torch.Tensor) -> None:
        if self.t.view(nat.DIAG_SLOTS, nat.DIAG_VALS)[:, 3].max().item() > 0:
            for f in fields:
                if not bool(torch.isfinite(torch.view_as_real(f) if f.is_complex() else f).all()):
                    _raise_divergence(step_index, f)
            _raise_divergence(step_index, fields[0])


def _grad_dot_r(R: _Real3, x_hat: torch.Tensor, v) -> torch.Tensor:
    """v . grad x = sum_i v_i F^-1(i d_i x_hat), real (hydro.py:83-85 order)."""
    g = R.grad_inv(x_hat)
    return _rpw(RPW_ADV3, v[0], g[0], v[1], g[1], v[2], g[2])


def _adv_term_r(R: _Real3, x_hat: torch.Tensor, axis: int, v_axis: torch.Tensor) -> torch.Tensor:
    """v_axis F^-1(i d_axis x_hat): one advection product (G = 8 helper roles)."""
    return _rpw(RPW_MUL, v_axis, R.inv(x_hat, deriv=axis))


def _density_r(R: _Real3, ph, ps, adv_hat, sym, hp: HydroParams, flag: _StepFlag, nl_hat=None,
               keep_z: bool = False, adv_pre_z: bool = False):
    """adv_hat = F(v . grad psi) (R.adv_fwd, or R.fwd of a physical sum;
    adv_pre_z: before its forward z pass); nl_hat = F(psi^3) when the caller
    has it (the previous step's mu), else transformed here up to its z pass,
    which the update runs (update_inv pre_z)."""
    nl_pre_z = nl_hat is None
    if nl_hat is None:
        nl_hat = R.fwd(ps, RPW_CUBE, z=False)
    return R.update_inv(0, ph, nl_hat, adv_hat, (float(sym.eps), float(hp.pfc.dt)), flag, keep_z=keep_z,
                        pre_z=(nl_pre_z, adv_pre_z))


def _density_mu_r(R: _Real3, ps, sym, want_nl: bool = False, grad_axes=None):
    """mu_hat = F(psi^3) + op F(psi) (hydro.py:99-101); the two forward z
    passes fused with the combination (pfcs_hydro_mu_z; PFCS_R2C_MUZ=0: the
    z passes and pfcs_hydro_mu separately, bit-identical).  want_nl: also
    return F(psi^3) — the next step's density update transforms the same
    psi**3 (hydro.py:86 after :99), so the serial steps carry it over."""
    nh, ny, nz = R.hshape
    kx, ky, kz = R.k
    nl_hat = R.fwd(ps, RPW_CUBE, z=not _R2C_MUZ)
    f_hat = R.fwd(ps, z=not _R2C_MUZ)
    st = nat.stream_ptr()
    if grad_axes and _R2C_MUZ and _R2C_MUZG and _R2C_GRAD and ny > 1 and 8 <= nz <= 4096 and nz & (nz - 1) == 0:
        # mu_hat never stored: the kernel runs grad mu's first inverse z passes
        # (the plain one for d_x / d_y, the i k_z one for d_z) — pfcs_hydro_mu_zgrad
        t0 = torch.empty_like(nl_hat) if any(a != 2 for a in grad_axes) else None
        tz = torch.empty_like(nl_hat) if 2 in grad_axes else None
        nl_out = torch.empty_like(nl_hat) if want_nl else None
        nat.call("pfcs_hydro_mu_zgrad", nat.ptr(nl_hat), nat.ptr(f_hat), None, nat.ptr(nl_out), nat.ptr(t0),
                 nat.ptr(tz), nat.ptr(R.d[2]), nh, ny, nz, nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), float(sym.eps), st)
        zpre = {"t0": t0, "tz": tz}
        return (None, nl_out, zpre) if want_nl else (None, zpre)
    mu = torch.empty_like(nl_hat)
    if _R2C_MUZ:
        nl_out = torch.empty_like(nl_hat) if want_nl else None
        nat.call("pfcs_hydro_mu_z", nat.ptr(nl_hat), nat.ptr(f_hat), nat.ptr(mu), nat.ptr(nl_out), nh, ny, nz,
                 nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), float(sym.eps), st)
    else:
        nat.call("pfcs_hydro_mu", nat.ptr(nl_hat), nat.ptr(f_hat), nat.ptr(mu), nh, ny, nz, nat.ptr(kx),
                 nat.ptr(ky), nat.ptr(kz), float(sym.eps), st)
        nl_out = nl_hat
    if grad_axes:
        return (mu, nl_out, None) if want_nl else (mu, None)
    return (mu, nl_out) if want_nl else mu


def _carry_slots(holder) -> dict:
    """Where a step keeps its carries: the fields object (serial steps) or a
    role-map rank's state dict."""
    return holder if isinstance(holder, dict) else holder.__dict__


def _z_carry_get(fields, key: str, h):
    """The {z, y} inverse passes of spectrum `h` kept by the previous step's
    update (update_inv keep_z), or None: valid only while `h` is still that
    step's state tensor, unmodified."""
    c = _carry_slots(fields).get("_pfcs_z", {}).get(key)
    if c is None or not _CARRY_NL:
        return None
    ref, version, z = c
    return z if (ref() is h and h._version == version) else None


def _z_carry_put(fields, key: str, h, z) -> None:
    d = _carry_slots(fields).setdefault("_pfcs_z", {})
    if isinstance(h, torch.Tensor) and z is not None and _CARRY_NL:
        d[key] = (weakref.ref(h), h._version, z)
    else:
        d.pop(key, None)


def _nl_carry_get(fields, ps):
    """F(psi^3) of `ps` carried over from the previous serial step (its mu),
    or None: valid only while fields.psi is still that step's tensor,
    unmodified (same object, same version counter)."""
    c = fields.__dict__.get("_pfcs_nl")
    if c is None or not _CARRY_NL:
        return None
    ref, version, nl = c
    return nl if (ref() is ps and ps._version == version) else None


def _nl_carry_put(fields, ps, nl) -> None:
    if isinstance(ps, torch.Tensor) and _CARRY_NL:
        fields.__dict__["_pfcs_nl"] = (weakref.ref(ps), ps._version, nl)
    else:
        fields.__dict__.pop("_pfcs_nl", None)


def _velocity_r(R: _Real3, vh, ps, axis: int, mu_hat, sym, hp: HydroParams, flag: _StepFlag, cc=None,
                muc=None, beta: float = 0.0, force=None, force_c=None, zpre=None):
    """force / force_c: F(psi F^-1(i d_axis mu_hat)) (/ c, muc) BEFORE their
    forward z pass (prod_grad z=False), when the caller formed all three at
    once (the serial steps); the update runs that z pass (pre_z)."""
    if force is None:
        force = R.prod_grad(mu_hat, ps, (axis,), z=False, zpre=zpre)[0]  # F(psi F^-1(i k mu_hat)), up to z
    if beta != 0.0:
        if force_c is None:
            force_c = R.prod_grad(muc, cc, (axis,), z=False)[0]
        total = torch.empty_like(force)
        nat.call("pfcs_axpy", nat.ptr(force), nat.ptr(force_c), nat.ptr(total), total.numel(), float(beta),
                 nat.stream_ptr())
        force = total
    dt, rho = float(hp.pfc.dt), float(hp.rho)
    return R.update_inv(1, vh, force, None, (dt / rho, (dt / rho) * float(hp.gamma), -0.5 * float(sym.a0) ** 2),
                        flag, pre_z=(True, False))


def _serial_hydro_step_r(fields: HydroFields, sym: SymbolTable, params: HydroParams) -> HydroFields:
    host = isinstance(fields.psi, np.ndarray)
    ps = _rdev(fields.psi)
    R = _Real3.of(ps.shape, sym, ps.device)
    flag = _StepFlag(ps.device)
    ph = _hdev(fields.psi_hat)
    vh = [_hdev(x) for x in fields.v_hat]
    _check_half(R, ph, *vh)
    vs = [_rdev(v) for v in fields.v]
    kpsi = _z_carry_get(fields, "psi", ph) or {}
    psi_hat, psi, zpsi = _density_r(R, ph, ps, R.adv_fwd(ph, vs, t0=kpsi.get("z"), y0=kpsi.get("y"), z=False), sym,
                                    params, flag, _nl_carry_get(fields, ps), keep_z=True, adv_pre_z=True)
    mu_hat, nl_next, zmu = _density_mu_r(R, psi, sym, want_nl=True, grad_axes=(0, 1, 2))  # shared by v_1..3
    forces = R.prod_grad(mu_hat, psi, z=False, zpre=zmu)
    out = [_velocity_r(R, vh[i], psi, i, mu_hat, sym, params, flag, force=forces[i]) for i in range(3)]
    flag.check(fields.step_index, psi_hat, *(o[0] for o in out))
    fields.psi_hat, fields.psi = _out(psi_hat, host), _out(psi, host)
    _nl_carry_put(fields, fields.psi, nl_next)
    _z_carry_put(fields, "psi", fields.psi_hat, zpsi)
    for i in range(3):
        fields.v_hat[i], fields.v[i] = _out(out[i][0], host), _out(out[i][1], host)
    fields.step_index += 1
    fields.sim_time += params.pfc.dt
    return fields


def _parallel_hydro_step_r(worker, role_state: dict, sym: SymbolTable, params: HydroParams) -> dict:
    """parallel_hydro_step on real device fields: psi and v_i travel as 8-byte
    real fields, the spectra are x-halved (bit-identical to the R2C serial step)."""
    rank = worker.rank
    psi0 = role_state["psi"]
    R = _Real3.of(tuple(psi0.shape), sym, psi0.device)
    flag = _StepFlag(psi0.device)
    idx = role_state["step_index"]
    worker.bcast_groups([(0, 1, 2, 3)])  # psi -> the velocity ranks: one broadcast (hydro.py:114-116)
    if rank == 0:
        ph = role_state["psi_hat"]
        _check_half(R, ph)
        kpsi = _z_carry_get(role_state, "psi", ph) or {}
        psi_hat, psi, zpsi = _density_r(R, ph, psi0, R.adv_fwd(ph, role_state["v"], t0=kpsi.get("z"),
                                                                y0=kpsi.get("y"), z=False),
                                        sym, params, flag, adv_pre_z=True, keep_z=True)
        _z_carry_put(role_state, "psi", psi_hat, zpsi)
        flag.check(idx, psi_hat)
        role_state["psi_hat"], role_state["psi"] = psi_hat, psi
        worker.bcast_tensor(0, (0, 1, 2, 3), TAG_PSI, t=psi)
        role_state["v"] = [worker.recv_tensor(i + 1, V_TAGS[i], torch.empty_like(psi)) for i in range(3)]
    else:
        i = rank - 1
        psi = worker.bcast_tensor(0, (0, 1, 2, 3), TAG_PSI, out=torch.empty_like(psi0))
        role_state["psi"] = psi
        _check_half(R, role_state["v_hat"])
        mu_hat, zmu = _density_mu_r(R, psi, sym, grad_axes=(i,))
        v_hat, v = _velocity_r(R, role_state["v_hat"], psi, i, mu_hat, sym, params, flag, zpre=zmu)
        flag.check(idx, v_hat)
        role_state["v_hat"], role_state["v_own"] = v_hat, v
        worker.send_tensor(0, V_TAGS[i], v)
    role_state["step_index"] = idx + 1
    return role_state
