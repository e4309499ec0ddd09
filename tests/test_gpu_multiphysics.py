"""Multiphysics field-per-GPU mode (density + composition + 3 velocities on
1, 5 or 8 workers).  No reference exists for the composition: the numpy
oracle restates the model (oracle/ref_numpy.py: multi_step).  With beta = 0
density and velocities must equal the reference's four-field dataflow."""

import math

import numpy as np
import pytest

from conftest import rel_inf

pytestmark = pytest.mark.gpu

EPS = -0.3


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_26818_b200 as p

    return p


def setup(pkg, n=16, beta=0.0, seed=3):
    from paper_2603_26818_b200.hydro import HydroParams
    from paper_2603_26818_b200.multiphysics import MultiFields, MultiParams
    from paper_2603_26818_b200.pfc import PfcParams, initial_field

    grid = pkg.GridSpec((n,) * 3, (2 * math.pi * math.sqrt(3),) * 3)
    hp = HydroParams(pfc=PfcParams(eps=EPS, dt=0.1), rho=1.0, gamma=1.0, a0=2.0)
    mp = MultiParams(hydro=hp, mobility=0.7, kappa=0.5, alpha=1.0, beta=beta)
    sym = pkg.make_symbols(grid, EPS, a0=2.0)
    psi0 = initial_field("two_mode_fcc_3d", grid, psi_bar=-0.3, amplitude=0.05)
    c0 = initial_field("constant_plus_noise", grid, psi_bar=0.0, seed=seed, noise_amplitude=0.1)
    psi_hat = np.fft.fftn(psi0.astype(np.complex128))
    c_hat = np.fft.fftn(c0.astype(np.complex128))
    rng = np.random.default_rng(seed)
    v = [(1e-3 * rng.standard_normal(grid.shape)).astype(np.complex128) for _ in range(3)]
    fields = MultiFields(psi_hat=psi_hat, psi=np.fft.ifftn(psi_hat), c_hat=c_hat, c=np.fft.ifftn(c_hat),
                         v_hat=[np.fft.fftn(x) for x in v], v=[x.copy() for x in v])
    return grid, sym, mp, fields


def copy_fields(f):
    from paper_2603_26818_b200.multiphysics import MultiFields

    return MultiFields(psi_hat=f.psi_hat.copy(), psi=f.psi.copy(), c_hat=f.c_hat.copy(), c=f.c.copy(),
                       v_hat=[x.copy() for x in f.v_hat], v=[x.copy() for x in f.v])


@pytest.mark.parametrize("beta", [0.0, 0.5])
def test_serial_vs_oracle(pkg, beta):
    import ref_numpy as ora
    from paper_2603_26818_b200.multiphysics import serial_multi_step

    grid, sym, mp, f = setup(pkg, beta=beta)
    o = {"psi_hat": f.psi_hat.copy(), "psi": f.psi.copy(), "c_hat": f.c_hat.copy(), "c": f.c.copy(),
         "v_hat": [x.copy() for x in f.v_hat], "v": [x.copy() for x in f.v]}
    osym = ora.symbols(grid.n, grid.length, EPS, a0=2.0)
    for _ in range(8):
        serial_multi_step(f, sym, mp)
        ora.multi_step(o, osym, 0.1, 1.0, 1.0, 0.7, 0.5, 1.0, beta)
    assert rel_inf(f.psi, o["psi"]) <= 1e-12
    assert rel_inf(f.c, o["c"]) <= 1e-12
    for i in range(3):
        assert rel_inf(f.v[i], o["v"][i]) <= 1e-9
    assert float(np.max(np.abs(f.c.imag))) <= 1e-12 * float(np.max(np.abs(f.c.real)))


def test_beta_zero_reproduces_four_field_hydro(pkg):
    from paper_2603_26818_b200.hydro import HydroFields, serial_hydro_step
    from paper_2603_26818_b200.multiphysics import serial_multi_step

    grid, sym, mp, f = setup(pkg)
    h = HydroFields(psi_hat=f.psi_hat.copy(), psi=f.psi.copy(), v_hat=[x.copy() for x in f.v_hat],
                    v=[x.copy() for x in f.v])
    for _ in range(5):
        serial_multi_step(f, sym, mp)
        serial_hydro_step(h, sym, mp.hydro)
    np.testing.assert_array_equal(f.psi_hat, h.psi_hat)
    for i in range(3):
        np.testing.assert_array_equal(f.v_hat[i], h.v_hat[i])


@pytest.mark.parametrize("G", [5, 8])
@pytest.mark.parametrize("beta", [0.0, 0.5])
def test_field_per_gpu_equals_serial_bitwise(pkg, G, beta):
    from paper_2603_26818_b200.multiphysics import (ROLES, initial_role_state, parallel_multi_step,
                                                    serial_multi_step)

    grid, sym, mp, f = setup(pkg, beta=beta)
    ref = copy_fields(f)
    for _ in range(4):
        serial_multi_step(ref, sym, mp)

    def body(w):
        st = initial_role_state(w.rank, G, f)
        for _ in range(4):
            parallel_multi_step(w, st, sym, mp)
        role = ROLES[G][w.rank]
        key = {"psi": "psi", "c": "c"}.get(role, "v_own")
        return role, st[key].cpu().numpy()

    for role, val in pkg.spawn_group(G, body):
        if role == "psi":
            np.testing.assert_array_equal(val, ref.psi)
        elif role == "c":
            np.testing.assert_array_equal(val, ref.c)
        elif role.startswith("v"):
            np.testing.assert_array_equal(val, ref.v[int(role[1]) - 1])
        else:  # adv helpers keep the latest v_i
            np.testing.assert_array_equal(val, ref.v[int(role[3]) - 1])


# ---------------------------------------------------------------- R2C path --

def to_real(f):
    """The same state as real physical fields + x-halved half spectra (the
    B200 R2C representation of multiphysics.py)."""
    from paper_2603_26818_b200.multiphysics import MultiFields

    def half(x):
        return np.fft.rfftn(np.real(x), axes=(1, 2, 0))

    return MultiFields(psi_hat=half(f.psi), psi=np.real(f.psi).copy(), c_hat=half(f.c), c=np.real(f.c).copy(),
                       v_hat=[half(x) for x in f.v], v=[np.real(x).copy() for x in f.v])


@pytest.mark.parametrize("beta", [0.0, 0.5])
def test_r2c_serial_vs_oracle(pkg, beta):
    """R2C path (real fields, half spectra) vs the complex oracle restatement:
    same tolerances as the C2C path."""
    import ref_numpy as ora
    from paper_2603_26818_b200.multiphysics import serial_multi_step

    grid, sym, mp, f = setup(pkg, beta=beta)
    o = {"psi_hat": f.psi_hat.copy(), "psi": f.psi.copy(), "c_hat": f.c_hat.copy(), "c": f.c.copy(),
         "v_hat": [x.copy() for x in f.v_hat], "v": [x.copy() for x in f.v]}
    r = to_real(f)
    osym = ora.symbols(grid.n, grid.length, EPS, a0=2.0)
    for _ in range(8):
        serial_multi_step(r, sym, mp)
        ora.multi_step(o, osym, 0.1, 1.0, 1.0, 0.7, 0.5, 1.0, beta)
    assert r.psi.dtype == np.float64 and r.psi_hat.shape == (9, 16, 16)
    assert rel_inf(r.psi, o["psi"].real) <= 1e-12
    assert rel_inf(r.c, o["c"].real) <= 1e-12
    for i in range(3):
        assert rel_inf(r.v[i], o["v"][i].real) <= 1e-9
    assert rel_inf(r.psi_hat, o["psi_hat"][:9]) <= 1e-12


def test_r2c_device_fields_and_c2c_agree(pkg):
    """Device-resident R2C fields (the hot path) vs the C2C path, 6 steps."""
    import torch
    from paper_2603_26818_b200.multiphysics import MultiFields, serial_multi_step

    grid, sym, mp, f = setup(pkg, n=32)
    r = to_real(f)
    d = MultiFields(psi_hat=torch.from_numpy(r.psi_hat).cuda(), psi=torch.from_numpy(r.psi).cuda(),
                    c_hat=torch.from_numpy(r.c_hat).cuda(), c=torch.from_numpy(r.c).cuda(),
                    v_hat=[torch.from_numpy(x).cuda() for x in r.v_hat], v=[torch.from_numpy(x).cuda() for x in r.v])
    for _ in range(6):
        serial_multi_step(d, sym, mp)
        serial_multi_step(f, sym, mp)
    assert d.psi.dtype == torch.float64 and d.psi.is_cuda
    assert rel_inf(d.psi.cpu().numpy(), f.psi.real) <= 1e-12
    assert rel_inf(d.c.cpu().numpy(), f.c.real) <= 1e-12
    for i in range(3):
        assert rel_inf(d.v[i].cpu().numpy(), f.v[i].real) <= 1e-9


@pytest.mark.parametrize("G", [5, 8])
@pytest.mark.parametrize("beta", [0.0, 0.5])
def test_r2c_field_per_gpu_equals_serial_bitwise(pkg, G, beta):
    from paper_2603_26818_b200.multiphysics import (ROLES, initial_role_state, parallel_multi_step,
                                                    serial_multi_step)

    grid, sym, mp, f0 = setup(pkg, beta=beta)
    f = to_real(f0)
    ref = to_real(f0)
    for _ in range(4):
        serial_multi_step(ref, sym, mp)

    def body(w):
        st = initial_role_state(w.rank, G, f)
        for _ in range(4):
            parallel_multi_step(w, st, sym, mp)
        role = ROLES[G][w.rank]
        key = {"psi": "psi", "c": "c"}.get(role, "v_own")
        return role, st[key].cpu().numpy()

    for role, val in pkg.spawn_group(G, body):
        assert val.dtype == np.float64
        if role == "psi":
            np.testing.assert_array_equal(val, ref.psi)
        elif role == "c":
            np.testing.assert_array_equal(val, ref.c)
        elif role.startswith("v"):
            np.testing.assert_array_equal(val, ref.v[int(role[1]) - 1])
        else:
            np.testing.assert_array_equal(val, ref.v[int(role[3]) - 1])


def test_r2c_divergence_raises(pkg):
    """A non-finite update raises DivergenceError at the step it happens
    (checked once per step on the R2C path)."""
    from paper_2603_26818_b200.multiphysics import serial_multi_step
    from paper_2603_26818_b200.pfc import DivergenceError

    grid, sym, mp, f = setup(pkg)
    r = to_real(f)
    r.psi = r.psi.copy()
    r.psi[3, 4, 5] = np.inf
    with pytest.raises(DivergenceError):
        serial_multi_step(r, sym, mp)


def test_r2c_rejects_full_grid_spectra(pkg):
    """Real physical fields with full-grid (C2C) spectra are a representation
    mix-up: the R2C path raises instead of computing on part of the array."""
    from paper_2603_26818_b200.hydro import HydroFields, serial_hydro_step
    from paper_2603_26818_b200.multiphysics import serial_multi_step

    grid, sym, mp, f = setup(pkg)
    r = to_real(f)
    r.psi_hat = f.psi_hat  # full complex spectrum next to a real psi
    with pytest.raises(ValueError, match="x-halved"):
        serial_multi_step(r, sym, mp)
    h = HydroFields(psi_hat=f.psi_hat, psi=np.real(f.psi).copy(), v_hat=[x for x in f.v_hat],
                    v=[np.real(x).copy() for x in f.v])
    with pytest.raises(ValueError, match="x-halved"):
        serial_hydro_step(h, sym, mp.hydro)


PRO_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import paper_2603_26818_b200 as pkg
from test_gpu_multiphysics import setup, to_real
from paper_2603_26818_b200.multiphysics import serial_multi_step
import torch
def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()
def host(x):
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else x
out = {{}}
for beta in (0.0, 0.5):
    grid, sym, mp, f = setup(pkg, n=32, beta=beta)
    r = to_real(f)
    if beta == 0.0:  # device-resident fields (the carried F(psi^3) applies to those)
        r.psi, r.c, r.psi_hat, r.c_hat = dev(r.psi), dev(r.c), dev(r.psi_hat), dev(r.c_hat)
        r.v, r.v_hat = [dev(x) for x in r.v], [dev(x) for x in r.v_hat]
    for k in range(4):
        serial_multi_step(r, sym, mp)
        if k == 1 and beta == 0.0:
            r.psi.mul_(1.0001)  # in-place edits must invalidate the carried F(psi^3) ...
            r.c_hat.mul_(1.0001)  # ... and the carried inverse z pass of c_hat
    for k in ("psi", "c", "psi_hat", "c_hat"):
        out[f"{{beta}}_{{k}}"] = host(getattr(r, k))
    for i in range(3):
        out[f"{{beta}}_v{{i}}"] = host(r.v[i])
np.savez({path!r}, **out)
"""


def test_r2c_fused_prologues_bit_identical(pkg, tmp_path):
    """The pointwise prologues fused into the R2C x pass (psi^3, psi * g,
    alpha (c^3 - c): pfcs_rfft_x_pro) and the psi / velocity / composition
    updates fused into the z pass of the following inverse
    (pfcs_update_zinv), the force products and the advection dot products
    in one fused x pass each (pfcs_xmul_x, pfcs_xdot3_x), the fused mu and
    the F(psi^3) carried from one step's mu to the next step's density update
    and the inverse z passes of psi_hat / c_hat carried from their updates to
    the next step's gradients (all invalidated by in-place edits) reproduce
    the unfused form (pfcs_real_pointwise +
    pfcs_rfft_x; the standalone update kernels + the plain inverse) bit for
    bit."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    here = Path(__file__).resolve().parent
    res = {}
    for flag in ("0", "1"):
        path = str(tmp_path / f"pro{flag}.npz")
        env = dict(os.environ, PFCS_R2C_PRO=flag, PFCS_R2C_UPD=flag, PFCS_R2C_XMUL=flag, PFCS_R2C_XDOT=flag,
                   PFCS_R2C_MUZ=flag, PFCS_R2C_CARRY=flag, PFCS_R2C_ZZ=flag,
                   PFCS_R2C_MUZG=flag)
        subprocess.run([sys.executable, "-c", PRO_CHILD.format(root=str(here.parent), tests=str(here), path=path)],
                       check=True, env=env, timeout=600)
        res[flag] = np.load(path)
    for k in res["0"].files:
        np.testing.assert_array_equal(res["0"][k], res["1"][k])


@pytest.mark.parametrize("G", [5, 8])
def test_r2c_production_fused_serial_equals_role_maps(pkg, G):
    """At 256^3 — where the fused advection / force x passes, the fused mu
    and the carries all take part (n = 16 runs their fallbacks) — the serial
    step on device fields (carries active) and the G = 5 / 8 role maps
    (no carries; G = 8 helpers form d_x x with pfcs_mul_deriv before a plain
    C2R) agree bit for bit after 3 steps."""
    import torch

    from paper_2603_26818_b200.multiphysics import ROLES, initial_role_state, parallel_multi_step, serial_multi_step

    grid, sym, mp, f0 = setup(pkg, n=256)
    f = to_real(f0)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    ref = to_real(f0)
    ref.psi, ref.c, ref.psi_hat, ref.c_hat = d(ref.psi), d(ref.c), d(ref.psi_hat), d(ref.c_hat)
    ref.v, ref.v_hat = [d(x) for x in ref.v], [d(x) for x in ref.v_hat]
    for _ in range(3):
        serial_multi_step(ref, sym, mp)
    want = {"psi": ref.psi.cpu().numpy(), "c": ref.c.cpu().numpy(), "v": [x.cpu().numpy() for x in ref.v]}
    del ref
    torch.cuda.empty_cache()

    def body(w):
        st = initial_role_state(w.rank, G, f)
        for _ in range(3):
            parallel_multi_step(w, st, sym, mp)
        role = ROLES[G][w.rank]
        key = {"psi": "psi", "c": "c"}.get(role, "v_own")
        return role, st[key].cpu().numpy()

    for role, val in pkg.spawn_group(G, body):
        if role in ("psi", "c"):
            np.testing.assert_array_equal(val, want[role])
        elif role.startswith("v"):
            np.testing.assert_array_equal(val, want["v"][int(role[1]) - 1])
        else:
            np.testing.assert_array_equal(val, want["v"][int(role[3]) - 1])


def test_r2c_production_one_step_vs_oracle(pkg):
    """One 256^3 serial step with every fused kernel of the production
    schedule (advection / force x passes, fused mu + grad mu z passes,
    updates with operand z passes) vs the complex oracle restatement."""
    import ref_numpy as ora
    from paper_2603_26818_b200.multiphysics import serial_multi_step

    grid, sym, mp, f = setup(pkg, n=256)
    o = {"psi_hat": f.psi_hat, "psi": f.psi, "c_hat": f.c_hat, "c": f.c, "v_hat": list(f.v_hat), "v": list(f.v)}
    r = to_real(f)
    osym = ora.symbols(grid.n, grid.length, EPS, a0=2.0)
    serial_multi_step(r, sym, mp)
    ora.multi_step(o, osym, 0.1, 1.0, 1.0, 0.7, 0.5, 1.0, 0.0)
    assert rel_inf(r.psi, o["psi"].real) <= 1e-12
    assert rel_inf(r.c, o["c"].real) <= 1e-12
    for i in range(3):
        assert rel_inf(r.v[i], o["v"][i].real) <= 1e-9
