"""CUDA parity of the hydrodynamic field-per-GPU mode (hydro.py:77-156)
against the reference's golden run, the numpy oracle and the reference's
own exactness tests."""

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


def fcc_grid(pkg, n):
    return pkg.GridSpec((n, n, n), (2 * math.pi * math.sqrt(3),) * 3)


def params(pkg, dt=0.1, rho=1.0, gamma=1.0, a0=1.0, psi_bar=-0.3):
    from paper_2603_26818_b200.hydro import HydroParams
    from paper_2603_26818_b200.pfc import PfcParams

    return HydroParams(pfc=PfcParams(eps=EPS, dt=dt, psi_bar=psi_bar, n_steps=1),
                       rho=rho, gamma=gamma, a0=a0)


def rand_complex(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def test_viscous_decay_bit_exact(pkg):
    from paper_2603_26818_b200.hydro import hydro_velocity_step

    grid = fcc_grid(pkg, 8)
    p = params(pkg, rho=1.3, gamma=0.7)
    sym = pkg.make_symbols(grid, EPS, a0=p.a0)
    psi = np.zeros(grid.shape, dtype=np.complex128)
    v_hat0 = rand_complex(grid.shape, 1)
    v_hat, _ = hydro_velocity_step(v_hat0.copy(), psi, sym.d1, sym, p)
    expected = v_hat0 / (1.0 - (p.pfc.dt / p.rho) * p.gamma * sym.lap)
    np.testing.assert_array_equal(v_hat, expected)


def test_velocity_matches_inline_reference(pkg):
    from paper_2603_26818_b200.hydro import hydro_velocity_step

    grid = fcc_grid(pkg, 16)
    p = params(pkg, rho=0.9, gamma=1.1, a0=2.0)
    sym = pkg.make_symbols(grid, EPS, a0=p.a0)
    rng = np.random.default_rng(3)
    psi = (0.05 * rng.standard_normal(grid.shape)).astype(np.complex128)
    v_hat0 = 0.01 * rand_complex(grid.shape, 4)
    got, _ = hydro_velocity_step(v_hat0.copy(), psi, sym.d3, sym, p)
    dt = p.pfc.dt
    mu_hat = np.fft.fftn(psi**3) + sym.op * np.fft.fftn(psi)
    force = np.fft.fftn(psi * np.fft.ifftn(sym.d3 * mu_hat))
    want = (v_hat0 - dt / p.rho * sym.cg * force) / (1.0 - dt / p.rho * p.gamma * sym.lap)
    assert rel_inf(got, want) <= 1e-12


def test_zero_velocity_reduces_to_pfc_bitwise(pkg):
    from paper_2603_26818_b200 import distfft
    from paper_2603_26818_b200.hydro import hydro_psi_step
    from paper_2603_26818_b200.pfc import PfcState, initial_field, pfc_step

    grid = fcc_grid(pkg, 8)
    p = params(pkg)
    psi0 = initial_field("two_mode_fcc_3d", grid, psi_bar=-0.3, amplitude=0.05, seed=0)
    sym = pkg.make_symbols(grid, EPS, a0=p.a0)
    zeros = np.zeros(grid.shape, dtype=np.complex128)
    psi_hat = pkg.fft_nd(psi0.astype(np.complex128))
    psi = pkg.fft_nd(psi_hat, forward=False)
    for _ in range(5):
        psi_hat, psi = hydro_psi_step(psi_hat, psi, zeros, zeros, zeros, sym, p)

    def body(w):
        f = distfft.scatter(psi0.astype(np.complex128), w, grid, distfft.Layout.Z_SLAB)
        st = PfcState(psi_hat=distfft.forward(f, w), grid=grid,
                      symbols=pkg.make_symbols(grid, EPS, layout=distfft.layout_for(
                          grid, distfft.Layout.X_SLAB, w.size), rank=w.rank), worker=w)
        for _ in range(5):
            pfc_step(st, p.pfc)
        return st.psi_hat.local

    np.testing.assert_array_equal(psi_hat, pkg.spawn_group(1, body)[0])


def test_advection_matches_inline_reference(pkg):
    from paper_2603_26818_b200.hydro import hydro_psi_step

    grid = pkg.GridSpec((16, 16, 16), (2 * math.pi,) * 3)
    p = params(pkg)
    sym = pkg.make_symbols(grid, EPS, a0=p.a0)
    x = np.arange(16) * (2 * math.pi / 16)
    psi = (np.cos(x)[:, None, None] * np.ones(grid.shape)).astype(np.complex128)
    psi_hat = np.fft.fftn(psi)
    v1 = np.full(grid.shape, 0.4, dtype=np.complex128)
    zeros = np.zeros_like(v1)
    got, _ = hydro_psi_step(psi_hat.copy(), psi, v1, zeros, zeros, sym, p)
    dt = p.pfc.dt
    adv = v1 * np.fft.ifftn(sym.d1 * psi_hat)
    want = (psi_hat + dt * (sym.lap * np.fft.fftn(psi**3) - np.fft.fftn(adv))) / (1.0 - dt * sym.linear)
    assert rel_inf(got, want) <= 1e-12


def _initial_fields(pkg, g, n):
    psi_hat = pkg.fft_nd(g["psi0"].astype(np.complex128))
    z = np.zeros((n,) * 3, dtype=np.complex128)
    return psi_hat, pkg.fft_nd(psi_hat, forward=False), z


def test_serial_hydro_vs_reference_golden(pkg, golden):
    from paper_2603_26818_b200.hydro import HydroFields, serial_hydro_step

    g = golden("hydro16")
    grid = fcc_grid(pkg, 16)
    p = params(pkg, a0=2.0)
    sym = pkg.make_symbols(grid, EPS, a0=2.0)
    psi_hat, psi, z = _initial_fields(pkg, g, 16)
    f = HydroFields(psi_hat=psi_hat, psi=psi, v_hat=[z.copy() for _ in range(3)],
                    v=[z.copy() for _ in range(3)])
    for _ in range(10):
        serial_hydro_step(f, sym, p)
    assert rel_inf(f.psi_hat, g["psi_hat"]) <= 1e-12
    assert rel_inf(f.psi, g["psi"]) <= 1e-12
    for i in range(3):
        assert rel_inf(f.v[i], g[f"v{i + 1}"]) <= 1e-9
        assert rel_inf(f.v_hat[i], g[f"vh{i + 1}"]) <= 1e-9


@pytest.mark.parametrize("device_msgs", [False, True])
def test_parallel_four_roles_equal_serial(pkg, golden, device_msgs):
    """Field-per-worker (G = 4) vs serial (G = 1) <= 1e-10 (acceptance:191-215)."""
    import torch

    from paper_2603_26818_b200.hydro import HydroFields, parallel_hydro_step, serial_hydro_step

    g = golden("hydro16")
    grid = fcc_grid(pkg, 16)
    p = params(pkg, a0=2.0)
    sym = pkg.make_symbols(grid, EPS, a0=2.0)
    psi_hat, psi, z = _initial_fields(pkg, g, 16)
    f = HydroFields(psi_hat=psi_hat.copy(), psi=psi.copy(), v_hat=[z.copy() for _ in range(3)],
                    v=[z.copy() for _ in range(3)])
    for _ in range(6):
        serial_hydro_step(f, sym, p)

    def conv(a):
        return torch.from_numpy(a).cuda() if device_msgs else a.copy()

    def body(w):
        if w.rank == 0:
            st = {"psi_hat": conv(psi_hat), "psi": conv(psi), "v": [conv(z) for _ in range(3)],
                  "step_index": 0}
        else:
            st = {"v_hat": conv(z), "psi": conv(z), "step_index": 0}
        for _ in range(6):
            parallel_hydro_step(w, st, sym, p)
        if w.rank == 0:
            return [np.asarray(st["psi"].cpu() if device_msgs else st["psi"])]
        return [np.asarray(st["v_own"].cpu() if device_msgs else st["v_own"])]

    res = pkg.spawn_group(4, body)
    assert rel_inf(res[0][0], f.psi) <= 1e-10
    for i in range(3):
        assert rel_inf(res[i + 1][0], f.v[i]) <= 1e-10


def test_gaussian_bump_width_adds_in_quadrature(pkg):
    n, L = 64, 40.0
    grid = pkg.GridSpec((n, n, n), (L,) * 3)
    s, a0 = 1.2, 1.5
    sym = pkg.make_symbols(grid, EPS, a0=a0)
    x = np.arange(n) * (L / n)
    c = L / 2
    r2 = ((x - c)[:, None, None] ** 2 + (x - c)[None, :, None] ** 2 + (x - c)[None, None, :] ** 2)
    bump = np.exp(-r2 / (2 * s**2)).astype(np.complex128)
    smooth = pkg.fft_nd(sym.cg * pkg.fft_nd(bump), forward=False).real
    second_moment = float(np.sum(r2 * smooth) / np.sum(smooth))
    assert second_moment == pytest.approx(3.0 * (s**2 + a0**2), rel=0.01)


def test_free_energy_full_matches_oracle(pkg):
    import ref_numpy as ora
    from paper_2603_26818_b200.hydro import free_energy_full

    grid = fcc_grid(pkg, 16)
    sym = pkg.make_symbols(grid, EPS, a0=2.0)
    rng = np.random.default_rng(9)
    psi = (-0.3 + 0.05 * rng.standard_normal(grid.shape)).astype(np.complex128)
    want = ora.free_energy(ora.fft_nd(psi), ora.symbols(grid.n, grid.length, EPS, 2.0), grid.cell_volume)
    assert free_energy_full(psi, sym, grid) == pytest.approx(want, rel=1e-12)


def _half(x):
    return np.fft.rfftn(np.real(x), axes=(1, 2, 0))


def test_serial_hydro_r2c_vs_reference_golden(pkg, golden):
    """Real fields (R2C path) vs the reference's 10-step golden run: same
    tolerances as the C2C path."""
    from paper_2603_26818_b200.hydro import HydroFields, serial_hydro_step

    g = golden("hydro16")
    grid = fcc_grid(pkg, 16)
    p = params(pkg, a0=2.0)
    sym = pkg.make_symbols(grid, EPS, a0=2.0)
    psi0 = np.real(g["psi0"]).astype(np.float64)
    z = np.zeros((16,) * 3)
    f = HydroFields(psi_hat=_half(psi0), psi=psi0.copy(), v_hat=[_half(z) for _ in range(3)],
                    v=[z.copy() for _ in range(3)])
    for _ in range(10):
        serial_hydro_step(f, sym, p)
    assert f.psi.dtype == np.float64 and f.psi_hat.shape == (9, 16, 16)
    assert rel_inf(f.psi, g["psi"].real) <= 1e-12
    assert rel_inf(f.psi_hat, g["psi_hat"][:9]) <= 1e-12
    for i in range(3):
        assert rel_inf(f.v[i], g[f"v{i + 1}"].real) <= 1e-9


def test_parallel_four_roles_r2c_equal_serial_bitwise(pkg, golden):
    import torch

    from paper_2603_26818_b200.hydro import HydroFields, parallel_hydro_step, serial_hydro_step

    g = golden("hydro16")
    grid = fcc_grid(pkg, 16)
    p = params(pkg, a0=2.0)
    sym = pkg.make_symbols(grid, EPS, a0=2.0)
    psi0 = np.real(g["psi0"]).astype(np.float64)
    z = np.zeros((16,) * 3)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    # device-resident serial fields: the serial steps carry F(psi^3) and the
    # psi update's inverse z pass between steps, the role map recomputes them
    f = HydroFields(psi_hat=d(_half(psi0)), psi=d(psi0), v_hat=[d(_half(z)) for _ in range(3)],
                    v=[d(z) for _ in range(3)])
    for _ in range(6):
        serial_hydro_step(f, sym, p)
    f.psi = f.psi.cpu().numpy()
    f.v = [x.cpu().numpy() for x in f.v]

    def body(w):
        if w.rank == 0:
            st = {"psi_hat": d(_half(psi0)), "psi": d(psi0), "v": [d(z) for _ in range(3)], "step_index": 0}
        else:
            st = {"v_hat": d(_half(z)), "psi": d(z), "step_index": 0}
        for _ in range(6):
            parallel_hydro_step(w, st, sym, p)
        return (st["psi"] if w.rank == 0 else st["v_own"]).cpu().numpy()

    res = pkg.spawn_group(4, body)
    np.testing.assert_array_equal(res[0], f.psi)
    for i in range(3):
        np.testing.assert_array_equal(res[i + 1], f.v[i])
