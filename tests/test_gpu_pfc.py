"""CUDA parity of the PFC stepper (pfc.py:96-182) against the reference's
golden runs and the numpy oracle, plus the reference's invariants.

Tolerances (north star): relative L2 <= 1e-9 on the field after 100 steps;
free energy non-increasing with 1e-9 slack (test_acceptance.py:128-129);
mean mode bit-invariant; constant state a bit-exact fixed point."""

import math

import numpy as np
import pytest

from conftest import rel_inf, rel_l2

pytestmark = pytest.mark.gpu

EPS = -0.3


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_26818_b200 as p

    return p


def make_state(pkg, w, grid, psi0, real=False, eps=EPS):
    from paper_2603_26818_b200 import distfft
    from paper_2603_26818_b200.pfc import PfcState

    xlay = distfft.layout_for(grid, distfft.Layout.X_SLAB, w.size)
    sym = pkg.make_symbols(grid, eps, layout=xlay, rank=w.rank)
    f = distfft.scatter(psi0 if real else psi0.astype(np.complex128), w, grid,
                        distfft.physical_layout(grid), real=real)
    return PfcState(psi_hat=distfft.forward(f, w), grid=grid, symbols=sym, worker=w)


def run_golden(pkg, golden_run, n, steps, G, real):
    from paper_2603_26818_b200 import distfft, pfc

    grid = pkg.GridSpec(n, tuple(golden_run["length"]))
    params = pfc.PfcParams(eps=EPS, dt=0.1, psi_bar=-0.3, n_steps=steps)

    def body(w):
        st = make_state(pkg, w, grid, golden_run["init"], real=real)
        energies = [pfc.free_energy(st, params)]
        means = [pfc.mean_and_max(st)]
        for s in range(steps):
            pfc.pfc_step(st, params)
            if (s + 1) % 20 == 0:
                energies.append(pfc.free_energy(st, params))
                means.append(pfc.mean_and_max(st))
        psi = distfft.gather(distfft.inverse(st.psi_hat, w), w)
        return np.real(psi), np.array(energies), np.array(means), st.last_max_imag_ratio

    return pkg.spawn_group(G, body)[0]


@pytest.mark.parametrize("real", [False, True])
@pytest.mark.parametrize("G", [1, 2, 4])
def test_pfc2d_256_100_steps_vs_reference(pkg, golden, real, G):
    """configs[0]: 2D PFC 256x256, 100 semi-implicit steps."""
    g = golden("pfc2d_256")
    psi, e, m, ratio = run_golden(pkg, g, (256, 256, 1), 100, G, real)
    assert rel_l2(psi, g["psi"]) <= 1e-9
    assert rel_inf(e, g["energies"]) <= 1e-9
    assert np.all(np.diff(e) <= 1e-9)
    assert m[0, 0] == m[-1, 0]  # mass bit-invariant
    assert rel_inf(m, g["means"]) <= 1e-9
    assert ratio <= 1e-10


@pytest.mark.parametrize("real", [False, True])
@pytest.mark.parametrize("G", [1, 2, 3])
def test_pfc3d_32_100_steps_vs_reference(pkg, golden, real, G):
    g = golden("pfc3d_32")
    psi, e, m, ratio = run_golden(pkg, g, (32, 32, 32), 100, G, real)
    assert rel_l2(psi, g["psi"]) <= 1e-9
    assert rel_inf(e, g["energies"]) <= 1e-9
    assert np.all(np.diff(e) <= 1e-9)
    assert len(set(m[:, 0])) == 1


@pytest.mark.parametrize("real", [False, True])
def test_pfc3d_fcc_vs_reference(pkg, golden, real):
    g = golden("pfc3d_fcc16")
    psi, e, m, _ = run_golden(pkg, g, (16, 16, 16), 40, 2, real)
    assert rel_l2(psi, g["psi"]) <= 1e-9
    assert rel_inf(e, g["energies"]) <= 1e-9


def test_uneven_grid_unfused_path(pkg):
    """10^3 on 3 workers (non-power-of-two: unfused kernels) vs the oracle."""
    import ref_numpy as ora
    from paper_2603_26818_b200 import distfft, pfc

    n = (10, 10, 10)
    grid = pkg.GridSpec(n, pfc.default_domain_length(n))
    psi0 = ora.initial_noise(n, seed=0)
    sym = ora.symbols(n, grid.length, EPS)
    want = ora.fft_nd(psi0.astype(np.complex128))
    for _ in range(20):
        want, _ = ora.pfc_step(want, sym, 0.1)
    params = pfc.PfcParams(n_steps=20)

    def body(w):
        st = make_state(pkg, w, grid, psi0)
        for _ in range(20):
            pfc.pfc_step(st, params)
        return distfft.gather(st.psi_hat, w)

    for G in (1, 3):
        got = pkg.spawn_group(G, body)[0]
        assert rel_inf(got, want) <= 1e-12


@pytest.mark.parametrize("real", [False, True])
def test_constant_state_is_fixed_point(pkg, real):
    from paper_2603_26818_b200.pfc import PfcParams, pfc_step

    grid = pkg.GridSpec((8, 8, 8), (2 * math.pi,) * 3)
    psi0 = np.full(grid.shape, -0.25)
    params = PfcParams(eps=EPS, dt=0.1, psi_bar=-0.25, n_steps=1)

    def body(w):
        st = make_state(pkg, w, grid, psi0, real=real)
        before = st.psi_hat.local.copy()
        pfc_step(st, params)
        np.testing.assert_array_equal(st.psi_hat.local, before)

    pkg.spawn_group(2, body)


def test_mean_mode_bit_invariant(pkg):
    from paper_2603_26818_b200.pfc import PfcParams, initial_field, pfc_step

    grid = pkg.GridSpec((8, 8, 8), (2 * math.pi,) * 3)
    psi0 = initial_field("constant_plus_noise", grid, psi_bar=-0.3, seed=7, noise_amplitude=0.05)
    params = PfcParams(n_steps=25)

    def body(w):
        st = make_state(pkg, w, grid, psi0)
        dc0 = st.psi_hat.local[0, 0, 0] if w.rank == 0 else None
        for _ in range(params.n_steps):
            pfc_step(st, params)
            if w.rank == 0:
                assert st.psi_hat.local[0, 0, 0] == dc0

    pkg.spawn_group(3, body)


@pytest.mark.parametrize("mode", [(1, 0, 0), (1, 1, 0), (1, 1, 1), (2, 1, 0), (3, 2, 1)])
def test_amplification_factor_law(pkg, mode):
    from paper_2603_26818_b200 import distfft
    from paper_2603_26818_b200.pfc import PfcParams, PfcState, pfc_step

    grid = pkg.GridSpec((16, 16, 16), (2 * math.pi,) * 3)
    dt, n = 0.1, 10
    k2 = float(sum(m**2 for m in mode))
    lin = -k2 * (EPS + (1 - k2) ** 2 * (4.0 / 3.0 - k2) ** 2)
    expected = 1e-10 * (1.0 / (1.0 - dt * lin)) ** n
    params = PfcParams(eps=EPS, dt=dt, psi_bar=0.0, n_steps=n)

    def body(w):
        spectrum = np.zeros(grid.shape, dtype=np.complex128)
        spectrum[mode] = 1e-10
        st = PfcState(psi_hat=distfft.scatter(spectrum, w, grid, distfft.Layout.X_SLAB,
                                              distfft.Space.SPECTRAL),
                      grid=grid,
                      symbols=pkg.make_symbols(grid, EPS, layout=distfft.layout_for(
                          grid, distfft.Layout.X_SLAB, w.size), rank=w.rank),
                      worker=w)
        for _ in range(n):
            pfc_step(st, params)
        return distfft.gather(st.psi_hat, w)

    amp = abs(pkg.spawn_group(2, body)[0][mode])
    assert amp == pytest.approx(expected, rel=1e-6)


def test_divergence_reports_step(pkg):
    from paper_2603_26818_b200.pfc import DivergenceError, PfcParams, pfc_step
    from paper_2603_26818_b200.transport import WorkerFailure

    grid = pkg.GridSpec((8, 8, 8), (2 * math.pi,) * 3)
    psi0 = np.full(grid.shape, 1e120)

    def body(w):
        st = make_state(pkg, w, grid, psi0)
        pfc_step(st, PfcParams(eps=EPS, dt=0.1, psi_bar=0.0, n_steps=1))

    with pytest.raises(WorkerFailure) as info:
        pkg.spawn_group(1, body)
    assert isinstance(info.value.cause, DivergenceError)
    assert info.value.cause.step_index == 0


def test_worker_count_invariance_bitwise(pkg):
    """Per-line arithmetic does not depend on G: G=1 and G=4 agree bit for bit."""
    from paper_2603_26818_b200 import distfft
    from paper_2603_26818_b200.pfc import PfcParams, initial_field, pfc_step

    grid = pkg.GridSpec((16, 16, 16), (2 * math.pi,) * 3)
    psi0 = initial_field("constant_plus_noise", grid, seed=5, noise_amplitude=0.05)

    for real in (False, True):
        def body(w):
            st = make_state(pkg, w, grid, psi0, real=real)
            for _ in range(30):
                pfc_step(st, PfcParams(n_steps=30))
            return distfft.gather(distfft.inverse(st.psi_hat, w), w)

        ref = pkg.spawn_group(1, body)[0]
        for G in (2, 4):
            np.testing.assert_array_equal(pkg.spawn_group(G, body)[0], ref)


def test_free_energy_closed_forms(pkg):
    from paper_2603_26818_b200.pfc import PfcParams, free_energy

    grid = pkg.GridSpec((16, 16, 16), (2 * math.pi,) * 3)
    A = 0.2
    x = np.arange(16) * (2 * math.pi / 16)
    psi0 = (A * np.cos(x))[:, None, None] * np.ones(grid.shape)
    expected = grid.volume * (A**2 / 4 * EPS + 3.0 / 32.0 * A**4)
    params = PfcParams(eps=EPS, dt=0.1, psi_bar=0.0, n_steps=1)

    for real in (False, True):
        def body(w):
            return free_energy(make_state(pkg, w, grid, psi0, real=real), params)

        vals = pkg.spawn_group(2, body)
        assert vals[0] == vals[1]
        assert vals[0] == pytest.approx(expected, rel=1e-10)


def test_r2c_matches_c2c_and_lean_oracle(pkg):
    """R2C state path vs the C2C path and the lean numpy R2C restatement."""
    import ref_numpy as ora
    from paper_2603_26818_b200 import distfft, pfc

    n = (64, 32, 16)
    grid = pkg.GridSpec(n, pfc.default_domain_length(n))
    psi0 = ora.initial_noise(n, seed=3, noise_amplitude=0.02)
    sym = ora.symbols(n, grid.length, EPS)
    half = np.fft.rfftn(psi0, axes=(1, 2, 0))
    for _ in range(50):
        half = ora.pfc_step_r2c(half, n, sym, 0.1)
    want = np.fft.irfftn(half, s=(n[1], n[2], n[0]), axes=(1, 2, 0))
    params = pfc.PfcParams(n_steps=50)

    def body(w):
        st = make_state(pkg, w, grid, psi0, real=True)
        for _ in range(50):
            pfc.pfc_step(st, params)
        return distfft.gather(distfft.inverse(st.psi_hat, w), w)

    got = pkg.spawn_group(2, body)[0]
    assert got.dtype == np.float64
    assert rel_l2(got, want) <= 1e-12


def test_pfc_run_graph_replay_matches_stepping(pkg):
    """pfc_run (CUDA-graph replay of 16-step blocks on one rank) is bit-identical
    to calling pfc_step, and reports divergence at the first bad step."""
    from paper_2603_26818_b200 import distfft, pfc

    n = (64, 64, 1)
    grid = pkg.GridSpec(n, pfc.default_domain_length(n))
    psi0 = pfc.initial_field("constant_plus_noise", grid, seed=3, noise_amplitude=0.02)
    params = pfc.PfcParams()

    def body(w):
        a = make_state(pkg, w, grid, psi0, real=True)
        b = make_state(pkg, w, grid, psi0, real=True)
        pfc.pfc_run(a, params, 50)
        for _ in range(50):
            pfc.pfc_step(b, params)
        pfc.pfc_run(a, params, 37)
        for _ in range(37):
            pfc.pfc_step(b, params)
        assert a.step_index == b.step_index == 87
        assert a.sim_time == b.sim_time
        return a.psi_hat.local, b.psi_hat.local

    x, y = pkg.spawn_group(1, body)[0]
    np.testing.assert_array_equal(x, y)

    def diverge(w):
        st = make_state(pkg, w, grid, np.full(grid.shape, 1e120), real=True)
        pfc.pfc_run(st, params, 40)

    with pytest.raises(Exception) as info:
        pkg.spawn_group(1, diverge)
    assert isinstance(info.value.cause, pfc.DivergenceError)
    assert info.value.cause.step_index == 0



@pytest.mark.parametrize("real", [True, False])
@pytest.mark.parametrize("n", [(32, 24, 32), (16, 12, 64)])
def test_peer_default_with_non_pow2_y(pkg, n, real):
    """Power-of-two x and z with a non-power-of-two y at G = 2 (default
    PFCS_EXCHANGE=peer): the fused y-line scatter only takes power-of-two y
    lines, so the engine must fall back to the collective exchange and stay
    bit-identical to G = 1."""
    from paper_2603_26818_b200 import distfft, pfc

    grid = pkg.GridSpec(n, pfc.default_domain_length(n))
    psi0 = pfc.initial_field("constant_plus_noise", grid, seed=4, noise_amplitude=0.05)

    def body(w):
        st = make_state(pkg, w, grid, psi0, real=real)
        pfc.pfc_run(st, pfc.PfcParams(), 5)
        return distfft.gather(st.psi_hat, w)

    ref = pkg.spawn_group(1, body)[0]
    got = pkg.spawn_group(2, body)[0]
    np.testing.assert_array_equal(got, ref)


def test_local_is_read_only_and_touch_invalidates(pkg):
    """DistField.local is a read-only host copy (an in-place edit would be
    silently lost, so it raises); editing .dev in place + touch() makes the
    PFC engine rebuild its prepared inverse."""
    from paper_2603_26818_b200 import distfft, pfc

    n = (16, 16, 16)
    grid = pkg.GridSpec(n, pfc.default_domain_length(n))
    psi0 = pfc.initial_field("constant_plus_noise", grid, seed=2, noise_amplitude=0.05)

    def body(w):
        st = make_state(pkg, w, grid, psi0, real=True)
        with pytest.raises(ValueError):
            st.psi_hat.local[0, 0, 0] = 1.0
        pfc.pfc_run(st, pfc.PfcParams(), 3)  # leaves a prepared inverse of psi_hat
        ref = make_state(pkg, w, grid, psi0, real=True)
        pfc.pfc_run(ref, pfc.PfcParams(), 3)
        # scale both in place: one through .dev + touch(), one by assignment
        st.psi_hat.dev.mul_(0.5)
        st.psi_hat.touch()
        ref.psi_hat.local = np.asarray(ref.psi_hat.local) * 0.5
        pfc.pfc_run(st, pfc.PfcParams(), 2)
        pfc.pfc_run(ref, pfc.PfcParams(), 2)
        return st.psi_hat.local.copy(), ref.psi_hat.local.copy()

    a, b = pkg.spawn_group(1, body)[0]
    np.testing.assert_array_equal(a, b)
