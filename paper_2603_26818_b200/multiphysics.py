"""Multiphysics PFC, field-per-GPU: density, composition and three velocity
components on 1, 5 or 8 GPUs (north-star item (3); BASELINE configs[4]).

The reference has the four-field hydrodynamic model on exactly 1 or 4
workers (hydro.py:1-15, hydro.py:129-156).  This module adds a composition
field c — Cahn-Hilliard, advected by the same velocity and optionally
feeding a Korteweg-type force back into it:

    mu_c  = alpha (c^3 - c) - kappa lap c
    dc/dt = M lap mu_c - v . grad c
    c_hat <- (c_hat + dt (M lap F[alpha (c^3 - c)] - F[v . grad c])) / (1 + dt M kappa lap^2)
    force_i = F[psi d_i mu_psi] + beta F[c d_i mu_c]

With beta = 0 (default) psi and v are bit-identical to the reference
four-field dataflow (hydro.serial_hydro_step) and c is a passive scalar.
There is no reference for c: oracle/ref_numpy.py restates these equations
(`multi_step`) and the tests check the GPU path against it.

Role maps (one field per GPU, rank -> role):
  G = 1: all roles serially (the oracle of the parallel modes)
  G = 5: 0 psi, 1..3 v1..v3, 4 c
  G = 8: as G = 5 plus 5..7 "advection" roles: rank 5+i computes
         v_i * F^-1(d_i psi_hat) concurrently with rank 0's F[psi^3], so the
         density step's critical path drops from 6 to 3 transforms.
Messages per step (device tensors; NCCL p2p between processes):
  psi_hat 0 -> 5,6,7 (tag 10, G=8) | products 5+i -> 0 (tag 11+i) |
  psi 0 -> 1,2,3 (tag 2) | c, c_hat 4 -> 1,2,3 (tags 7, 8; beta != 0) |
  v_i 1+i -> 0, 4 (tags 4,5,6) and -> 5+i (G=8).
All modes produce bit-identical fields (same kernels, same summation order).

Representations.  Complex full-grid fields (the reference's own
representation, hydro.py:60-69) take the C2C path below.  Real physical
fields (psi, c, v_i float64) select the B200 R2C path (`_Real3`): spectra
are x-halved (n/2+1, n, n) half spectra, every transform is rfft_x / irfft_x
plus the y and z C2C passes (R + 5S bytes instead of 6C: half the HBM
traffic), the pointwise products and nonlinearities read and write 8-byte
real samples (pfcs_real_pointwise), the derivative multipliers stay fused
into the first pass of the inverse transforms, and the non-finite checks of
a step are collected in one device flag read back once per step instead of
one host round trip per spectral update.  The R2C results equal the C2C
ones to rounding (<= 1e-12, oracle/ref_numpy.py:multi_step) and the serial
and field-per-GPU R2C modes are bit-identical to each other.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dataclass_field

import numpy as np
import torch

from . import _native as nat
from .grid import SymbolTable
from .hydro import (HydroParams, TAG_PSI, V_TAGS, RPW_ADD3, RPW_CHNL, _check_half, _dev, _Diag, _Real3, _StepFlag,
                    _adv_term_r, _density_mu_r, _density_r, _fft, _fft_cmul, _fft_cube, _hdev, _ifft_deriv,
                    _is_real, _nl_carry_get, _nl_carry_put, _out, _raise_divergence, _rdev, _rpw, _vectors,
                    _velocity_r, _z_carry_get, _z_carry_put)

__all__ = [
    "MultiParams",
    "MultiFields",
    "ROLES",
    "composition_step",
    "density_step",
    "velocity_step",
    "serial_multi_step",
    "parallel_multi_step",
    "initial_role_state",
]

TAG_C = 7
TAG_CHAT = 8
TAG_PSIHAT = 10
ADV_TAGS = (11, 12, 13)

ROLES = {
    1: ["all"],
    5: ["psi", "v1", "v2", "v3", "c"],
    8: ["psi", "v1", "v2", "v3", "c", "adv1", "adv2", "adv3"],
}


@dataclass
class MultiParams:
    hydro: HydroParams = dataclass_field(default_factory=HydroParams)
    mobility: float = 1.0
    kappa: float = 1.0
    alpha: float = 1.0
    beta: float = 0.0

    def __post_init__(self):
        if not (self.mobility > 0 and self.kappa >= 0):
            raise ValueError("mobility must be > 0 and kappa >= 0")


@dataclass
class MultiFields:
    psi_hat: object
    psi: object
    c_hat: object
    c: object
    v_hat: list
    v: list
    step_index: int = 0
    sim_time: float = 0.0


def _st():
    return nat.stream_ptr()


def _adv_product(x_hat: torch.Tensor, axis: int, v: torch.Tensor, sym) -> torch.Tensor:
    """v_axis * F^-1(d_axis * x_hat) (one term of v . grad x)."""
    g = _ifft_deriv(x_hat, axis, sym)
    p = torch.empty_like(g)
    nat.call("pfcs_cmul", nat.ptr(v), nat.ptr(g), nat.ptr(p), p.numel(), _st())
    return p


def _sum3(a, b, c):
    out = torch.empty_like(a)
    nat.call("pfcs_add3", nat.ptr(a), nat.ptr(b), nat.ptr(c), nat.ptr(out), out.numel(), _st())
    return out


def density_step(psi_hat, psi, products, sym: SymbolTable, params: MultiParams, step_index=0):
    """psi update (hydro.py:77-90) from the three advection products
    v_i * F^-1(d_i psi_hat) (computed here or by the adv roles)."""
    ph, ps = _dev(psi_hat), _dev(psi)
    dev = ph.device
    kx, ky, kz = _vectors(sym, dev)[:3]
    n0, n1, n2 = ph.shape
    nl_hat = _fft_cube(ps)
    adv_hat = _fft(_sum3(*products), True)
    new = torch.empty_like(ph)
    diag = _Diag(dev)
    nat.call("pfcs_hydro_psi_update_to", nat.ptr(ph), nat.ptr(new), nat.ptr(nl_hat), nat.ptr(adv_hat), n0, n1, n2,
             nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), float(sym.eps), float(params.hydro.pfc.dt),
             nat.ptr(diag.t), _st())
    if diag.bad():
        _raise_divergence(step_index, new)
    return new, _fft(new, False)


def composition_step(c_hat, c, v, sym: SymbolTable, params: MultiParams, step_index=0):
    """Advected Cahn-Hilliard update of the composition (see module doc)."""
    ch, cc = _dev(c_hat), _dev(c)
    vs = [_dev(x) for x in v]
    dev = ch.device
    kx, ky, kz = _vectors(sym, dev)[:3]
    n0, n1, n2 = ch.shape
    prods = [_adv_product(ch, i, vs[i], sym) for i in range(3)]
    adv_hat = _fft(_sum3(*prods), True)
    del prods
    f = torch.empty_like(cc)
    nat.call("pfcs_ch_nonlin", nat.ptr(cc), nat.ptr(f), f.numel(), float(params.alpha), _st())
    f_hat = _fft(f, True)
    new = torch.empty_like(ch)
    diag = _Diag(dev)
    nat.call("pfcs_ch_update_to", nat.ptr(ch), nat.ptr(new), nat.ptr(f_hat), nat.ptr(adv_hat), n0, n1, n2, nat.ptr(kx),
             nat.ptr(ky), nat.ptr(kz), float(params.mobility), float(params.kappa),
             float(params.hydro.pfc.dt), nat.ptr(diag.t), _st())
    if diag.bad():
        _raise_divergence(step_index, new)
    return new, _fft(new, False)


def density_mu(psi, sym: SymbolTable) -> torch.Tensor:
    """mu_hat = F[psi^3] + op F[psi] (hydro.py:96-97): the chemical potential
    every velocity component's force is built from."""
    ps = _dev(psi)
    kx, ky, kz = _vectors(sym, ps.device)[:3]
    n0, n1, n2 = ps.shape
    nl_hat = _fft_cube(ps)
    f_hat = _fft(ps, True)
    mu_hat = torch.empty_like(ps)
    nat.call("pfcs_hydro_mu", nat.ptr(nl_hat), nat.ptr(f_hat), nat.ptr(mu_hat), n0, n1, n2, nat.ptr(kx),
             nat.ptr(ky), nat.ptr(kz), float(sym.eps), _st())
    return mu_hat


def composition_mu(c, c_hat, sym: SymbolTable, params: MultiParams) -> torch.Tensor:
    """mu_c = F[f'(c)] + kappa k^2 c_hat, the composition force's potential."""
    cc, chh = _dev(c), _dev(c_hat)
    kx, ky, kz = _vectors(sym, cc.device)[:3]
    n0, n1, n2 = cc.shape
    st = _st()
    fc = torch.empty_like(cc)
    nat.call("pfcs_ch_nonlin", nat.ptr(cc), nat.ptr(fc), fc.numel(), float(params.alpha), st)
    fc_hat = _fft(fc, True)
    muc = torch.empty_like(fc_hat)
    nat.call("pfcs_ch_mu", nat.ptr(fc_hat), nat.ptr(chh), nat.ptr(muc), n0, n1, n2, nat.ptr(kx), nat.ptr(ky),
             nat.ptr(kz), float(params.kappa), st)
    return muc


def velocity_step(v_hat, psi, axis: int, sym: SymbolTable, params: MultiParams, c=None, c_hat=None,
                  step_index=0, *, mu_hat=None, mu_c=None):
    """hydro_velocity_step (hydro.py:93-107) plus beta * F[c d_axis mu_c].
    ``mu_hat`` / ``mu_c`` (from density_mu / composition_mu) may be passed in
    when several components are advanced from the same fields (serial mode
    computes them once per step instead of once per component)."""
    vh, ps = _dev(v_hat), _dev(psi)
    dev = vh.device
    kx, ky, kz = _vectors(sym, dev)[:3]
    n0, n1, n2 = vh.shape
    st = _st()
    if mu_hat is None:
        mu_hat = density_mu(ps, sym)
    force = _fft_cmul(ps, _ifft_deriv(mu_hat, axis, sym))  # F(psi * F^-1(i k mu_hat)), both fused
    if params.beta != 0.0:
        cc = _dev(c)
        muc = mu_c if mu_c is not None else composition_mu(cc, c_hat, sym, params)
        force_c = _fft_cmul(cc, _ifft_deriv(muc, axis, sym))
        total = torch.empty_like(force)
        nat.call("pfcs_axpy", nat.ptr(force), nat.ptr(force_c), nat.ptr(total), total.numel(),
                 float(params.beta), st)
        force = total
    hp = params.hydro
    dt, rho = float(hp.pfc.dt), float(hp.rho)
    new = torch.empty_like(vh)
    diag = _Diag(dev)
    nat.call("pfcs_hydro_vel_update_to", nat.ptr(vh), nat.ptr(new), nat.ptr(force), n0, n1, n2, nat.ptr(kx), nat.ptr(ky),
             nat.ptr(kz), dt / rho, (dt / rho) * float(hp.gamma), -0.5 * float(sym.a0) ** 2,
             nat.ptr(diag.t), st)
    if diag.bad():
        _raise_divergence(step_index, new)
    return new, _fft(new, False)


def serial_multi_step(fields: MultiFields, sym: SymbolTable, params: MultiParams) -> MultiFields:
    """All five roles on one GPU: density and composition from the previous
    velocities, then the velocities from the fresh density (and composition).
    Real physical fields take the R2C path (module doc)."""
    if _is_real(fields.psi):
        return _serial_multi_step_r(fields, sym, params)
    host = isinstance(fields.psi_hat, np.ndarray)
    ph = _dev(fields.psi_hat)
    vs = [_dev(v) for v in fields.v]
    prods = [_adv_product(ph, i, vs[i], sym) for i in range(3)]
    psi_hat, psi = density_step(ph, fields.psi, prods, sym, params, fields.step_index)
    del prods
    c_hat, c = composition_step(fields.c_hat, fields.c, vs, sym, params, fields.step_index)
    # the three components share mu_hat (and mu_c): computed once
    mu_hat = density_mu(psi, sym)
    mu_c = composition_mu(c, c_hat, sym, params) if params.beta != 0.0 else None
    for i in range(3):
        vh, v = velocity_step(fields.v_hat[i], psi, i, sym, params, c=c, c_hat=c_hat,
                              step_index=fields.step_index, mu_hat=mu_hat, mu_c=mu_c)
        fields.v_hat[i], fields.v[i] = _out(vh, host), _out(v, host)
    fields.psi_hat, fields.psi = _out(psi_hat, host), _out(psi, host)
    fields.c_hat, fields.c = _out(c_hat, host), _out(c, host)
    fields.step_index += 1
    fields.sim_time += params.hydro.pfc.dt
    return fields


def initial_role_state(rank: int, G: int, fields: MultiFields) -> dict:
    """The slice of a MultiFields a rank owns in the G-role map (device)."""
    role = ROLES[G][rank]
    real = _is_real(fields.psi)
    st = {"step_index": fields.step_index, "role": role, "real": real}
    phys = _rdev if real else _dev  # physical fields: real (R2C path) or complex (C2C)
    if role == "psi":
        st.update(psi_hat=_dev(fields.psi_hat), psi=phys(fields.psi), v=[phys(v) for v in fields.v])
    elif role == "c":
        st.update(c_hat=_dev(fields.c_hat), c=phys(fields.c), v=[phys(v) for v in fields.v])
    elif role.startswith("v"):
        i = int(role[1]) - 1
        st.update(v_hat=_dev(fields.v_hat[i]), v_own=phys(fields.v[i]), psi=phys(fields.psi),
                  c=phys(fields.c), c_hat=_dev(fields.c_hat))
    elif role.startswith("adv"):
        i = int(role[3]) - 1
        st.update(v_own=phys(fields.v[i]), psi_hat=_dev(fields.psi_hat))
    return st


def parallel_multi_step(worker, st: dict, sym: SymbolTable, params: MultiParams) -> dict:
    """One step of the field-per-GPU dataflow (G = 5 or 8, see module doc)."""
    G = worker.size
    if G not in (5, 8):
        raise ValueError(f"multiphysics field-per-GPU mode runs on 5 or 8 workers, got {G}")
    if st.get("real"):
        return _parallel_multi_step_r(worker, st, sym, params)
    role = ROLES[G][worker.rank]
    idx = st["step_index"]
    beta = params.beta != 0.0
    if role == "psi":
        ph = st["psi_hat"]
        if G == 8:
            for h in (5, 6, 7):
                worker.send_tensor(h, TAG_PSIHAT, ph)
            prods = [worker.recv_tensor(5 + i, ADV_TAGS[i], torch.empty_like(ph)) for i in range(3)]
        else:
            prods = [_adv_product(ph, i, st["v"][i], sym) for i in range(3)]
        st["psi_hat"], st["psi"] = density_step(ph, st["psi"], prods, sym, params, idx)
        for dst in (1, 2, 3):
            worker.send_tensor(dst, TAG_PSI, st["psi"])
        st["v"] = [worker.recv_tensor(1 + i, V_TAGS[i], torch.empty_like(ph)) for i in range(3)]
    elif role == "c":
        st["c_hat"], st["c"] = composition_step(st["c_hat"], st["c"], st["v"], sym, params, idx)
        if beta:
            for dst in (1, 2, 3):
                worker.send_tensor(dst, TAG_C, st["c"])
                worker.send_tensor(dst, TAG_CHAT, st["c_hat"])
        st["v"] = [worker.recv_tensor(1 + i, V_TAGS[i], torch.empty_like(st["c"])) for i in range(3)]
    elif role.startswith("v"):
        i = int(role[1]) - 1
        psi = worker.recv_tensor(0, TAG_PSI, torch.empty_like(st["psi"]))
        st["psi"] = psi
        if beta:
            st["c"] = worker.recv_tensor(4, TAG_C, torch.empty_like(st["c"]))
            st["c_hat"] = worker.recv_tensor(4, TAG_CHAT, torch.empty_like(st["c_hat"]))
        st["v_hat"], st["v_own"] = velocity_step(st["v_hat"], psi, i, sym, params, c=st.get("c"),
                                                 c_hat=st.get("c_hat"), step_index=idx)
        dsts = (0, 4) + ((5 + i,) if G == 8 else ())
        for dst in dsts:
            worker.send_tensor(dst, V_TAGS[i], st["v_own"])
    else:  # advection helper (G = 8)
        i = int(role[3]) - 1
        ph = worker.recv_tensor(0, TAG_PSIHAT, torch.empty_like(st["psi_hat"]))
        worker.send_tensor(0, ADV_TAGS[i], _adv_product(ph, i, st["v_own"], sym))
        st["v_own"] = worker.recv_tensor(1 + i, V_TAGS[i], torch.empty_like(ph))
    st["step_index"] = idx + 1
    return st


# ------------------------------------------------------------ R2C path ------

def _composition_r(R: _Real3, ch, cc, v, sym, params: MultiParams, flag: _StepFlag, t0=None, keep_z=False,
                   y0=None):
    """t0 / y0: the plain inverse z / z + y passes of ch if the caller has
    them; keep_z: also return the new state's (update_inv)."""
    adv_hat = R.adv_fwd(ch, v, t0=t0, y0=y0, z=False)
    f_hat = R.fwd(cc, RPW_CHNL, alpha=params.alpha, z=False)
    return R.update_inv(2, ch, f_hat, adv_hat,
                        (float(params.mobility), float(params.kappa), float(params.hydro.pfc.dt)), flag,
                        keep_z=keep_z, pre_z=(True, True))


def _composition_mu_r(R: _Real3, cc, ch, params: MultiParams) -> torch.Tensor:
    nh, ny, nz = R.hshape
    kx, ky, kz = R.k
    fc_hat = R.fwd(cc, RPW_CHNL, alpha=params.alpha)
    muc = torch.empty_like(fc_hat)
    nat.call("pfcs_ch_mu", nat.ptr(fc_hat), nat.ptr(ch), nat.ptr(muc), nh, ny, nz, nat.ptr(kx), nat.ptr(ky),
             nat.ptr(kz), float(params.kappa), _st())
    return muc


def _serial_multi_step_r(fields: MultiFields, sym: SymbolTable, params: MultiParams) -> MultiFields:
    host = isinstance(fields.psi, np.ndarray)
    ps = _rdev(fields.psi)
    R = _Real3.of(ps.shape, sym, ps.device)
    flag = _StepFlag(ps.device)
    ph, ch, cc = _hdev(fields.psi_hat), _hdev(fields.c_hat), _rdev(fields.c)
    vh = [_hdev(x) for x in fields.v_hat]
    _check_half(R, ph, ch, *vh)
    vs = [_rdev(v) for v in fields.v]
    kpsi = _z_carry_get(fields, "psi", ph) or {}
    kc = _z_carry_get(fields, "c", ch) or {}
    psi_hat, psi, zpsi = _density_r(R, ph, ps, R.adv_fwd(ph, vs, t0=kpsi.get("z"), y0=kpsi.get("y"), z=False), sym,
                                    params.hydro, flag, _nl_carry_get(fields, ps), keep_z=True, adv_pre_z=True)
    c_hat, c, zc = _composition_r(R, ch, cc, vs, sym, params, flag, t0=kc.get("z"), y0=kc.get("y"), keep_z=True)
    mu_hat, nl_next, zmu = _density_mu_r(R, psi, sym, want_nl=True, grad_axes=(0, 1, 2))
    muc = _composition_mu_r(R, c, c_hat, params) if params.beta != 0.0 else None
    forces = R.prod_grad(mu_hat, psi, z=False, zpre=zmu)
    forces_c = R.prod_grad(muc, c, z=False) if muc is not None else [None] * 3
    out = [_velocity_r(R, vh[i], psi, i, mu_hat, sym, params.hydro, flag, c, muc, params.beta, forces[i],
                       forces_c[i]) for i in range(3)]
    flag.check(fields.step_index, psi_hat, c_hat, *(o[0] for o in out))
    for i in range(3):
        fields.v_hat[i], fields.v[i] = _out(out[i][0], host), _out(out[i][1], host)
    fields.psi_hat, fields.psi = _out(psi_hat, host), _out(psi, host)
    _nl_carry_put(fields, fields.psi, nl_next)
    _z_carry_put(fields, "psi", fields.psi_hat, zpsi)
    fields.c_hat, fields.c = _out(c_hat, host), _out(c, host)
    _z_carry_put(fields, "c", fields.c_hat, zc)
    fields.step_index += 1
    fields.sim_time += params.hydro.pfc.dt
    return fields


def _parallel_multi_step_r(worker, st: dict, sym: SymbolTable, params: MultiParams) -> dict:
    """The G = 5 / 8 dataflow of parallel_multi_step on real fields: the
    messages are real physical fields (8 bytes per point) and half spectra."""
    G = worker.size
    role = ROLES[G][worker.rank]
    idx = st["step_index"]
    beta = params.beta != 0.0
    like = st.get("psi") if st.get("psi") is not None else st.get("c", st.get("v_own"))
    R = _Real3.of(tuple(like.shape), sym, like.device)
    _check_half(R, *(st[k] for k in ("psi_hat", "c_hat", "v_hat") if k in st))
    flag = _StepFlag(like.device)
    # one-to-many messages as broadcasts over fixed rank sets (declared
    # collectively, in the same order, on every rank)
    s_psi, s_psih, s_c = (0, 1, 2, 3), (0, 5, 6, 7), (1, 2, 3, 4)
    s_v = [(0, 1 + i, 4) + ((5 + i,) if G == 8 else ()) for i in range(3)]
    worker.bcast_groups([s_psi, *s_v] + ([s_psih] if G == 8 else []) + ([s_c] if beta else []))
    if role == "psi":
        ph = st["psi_hat"]
        if G == 8:
            worker.bcast_tensor(0, s_psih, TAG_PSIHAT, t=ph)
            p = [worker.recv_tensor(5 + i, ADV_TAGS[i], torch.empty_like(st["psi"])) for i in range(3)]
            adv_hat = R.fwd(_rpw(RPW_ADD3, *p), z=False)
        else:  # (the rank's previous update kept ph's inverse z / y passes)
            kpsi = _z_carry_get(st, "psi", ph) or {}
            adv_hat = R.adv_fwd(ph, st["v"], t0=kpsi.get("z"), y0=kpsi.get("y"), z=False)
        st["psi_hat"], st["psi"], zpsi = _density_r(R, ph, st["psi"], adv_hat, sym, params.hydro, flag,
                                                    adv_pre_z=True, keep_z=True)
        _z_carry_put(st, "psi", st["psi_hat"], zpsi if G != 8 else None)  # (G = 8: the helpers form grad psi)
        flag.check(idx, st["psi_hat"])
        worker.bcast_tensor(0, s_psi, TAG_PSI, t=st["psi"])
        st["v"] = [worker.bcast_tensor(1 + i, s_v[i], V_TAGS[i], out=torch.empty_like(st["psi"]))
                   for i in range(3)]
    elif role == "c":
        kc = _z_carry_get(st, "c", st["c_hat"]) or {}
        st["c_hat"], st["c"], zc = _composition_r(R, st["c_hat"], st["c"], st["v"], sym, params, flag,
                                                  t0=kc.get("z"), y0=kc.get("y"), keep_z=True)
        _z_carry_put(st, "c", st["c_hat"], zc)
        flag.check(idx, st["c_hat"])
        if beta:
            worker.bcast_tensor(4, s_c, TAG_C, t=st["c"])
            worker.bcast_tensor(4, s_c, TAG_CHAT, t=st["c_hat"])
        st["v"] = [worker.bcast_tensor(1 + i, s_v[i], V_TAGS[i], out=torch.empty_like(st["c"])) for i in range(3)]
    elif role.startswith("v"):
        i = int(role[1]) - 1
        psi = worker.bcast_tensor(0, s_psi, TAG_PSI, out=torch.empty_like(st["psi"]))
        st["psi"] = psi
        muc = None
        if beta:
            st["c"] = worker.bcast_tensor(4, s_c, TAG_C, out=torch.empty_like(st["c"]))
            st["c_hat"] = worker.bcast_tensor(4, s_c, TAG_CHAT, out=torch.empty_like(st["c_hat"]))
            muc = _composition_mu_r(R, st["c"], st["c_hat"], params)
        mu_hat, zmu = _density_mu_r(R, psi, sym, grad_axes=(i,))
        st["v_hat"], st["v_own"] = _velocity_r(R, st["v_hat"], psi, i, mu_hat, sym, params.hydro, flag, st.get("c"),
                                                muc, params.beta, zpre=zmu)
        flag.check(idx, st["v_hat"])
        worker.bcast_tensor(1 + i, s_v[i], V_TAGS[i], t=st["v_own"])
    else:  # advection helper (G = 8)
        i = int(role[3]) - 1
        ph = worker.bcast_tensor(0, s_psih, TAG_PSIHAT, out=torch.empty_like(st["psi_hat"]))
        worker.send_tensor(0, ADV_TAGS[i], _adv_term_r(R, ph, i, st["v_own"]))
        st["v_own"] = worker.bcast_tensor(1 + i, s_v[i], V_TAGS[i], out=torch.empty_like(st["v_own"]))
    st["step_index"] = idx + 1
    return st
