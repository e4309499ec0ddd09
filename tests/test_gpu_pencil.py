"""Pencil decomposition (new; no reference counterpart): parity of the
distributed transform against numpy's fftn and of the PFC step against the
slab path (bit-identical: per-line arithmetic does not depend on the
decomposition) and against the reference's golden run."""

import numpy as np
import pytest

from conftest import rel_inf, rel_l2

pytestmark = pytest.mark.gpu

GRIDS = [(1, 1), (1, 2), (2, 1), (2, 2), (2, 3), (2, 4)]


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_26818_b200 as p

    return p


def _roundtrip(pkg, x, pr, pc, real):
    from paper_2603_26818_b200 import distfft
    from paper_2603_26818_b200.pencil import PencilGrid, pencil_scatter

    grid = pkg.GridSpec(x.shape, (1.0, 1.0, 1.0))
    pg = PencilGrid(pr, pc)

    def body(w):
        f = pencil_scatter(x, w, grid, pg, real=real)
        spec = distfft.forward(f, w)
        back = distfft.inverse(spec, w)
        return distfft.gather(spec, w), distfft.gather(back, w)

    return pkg.spawn_group(pr * pc, body)


@pytest.mark.parametrize("shape", [(8, 12, 16), (16, 16, 16), (32, 16, 8), (6, 10, 7), (4, 4, 2)])
@pytest.mark.parametrize("pr,pc", GRIDS)
def test_pencil_c2c(pkg, shape, pr, pc):
    rng = np.random.default_rng(5)
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    for spec, back in _roundtrip(pkg, x, pr, pc, False):
        assert rel_inf(spec, np.fft.fftn(x)) <= 1e-12
        assert rel_inf(back, x) <= 1e-12


@pytest.mark.parametrize("shape", [(8, 12, 16), (16, 16, 16), (64, 32, 16), (4, 8, 8)])
@pytest.mark.parametrize("pr,pc", GRIDS)
def test_pencil_r2c(pkg, shape, pr, pc):
    x = np.random.default_rng(6).standard_normal(shape)
    for spec, back in _roundtrip(pkg, x, pr, pc, True):
        assert rel_inf(spec, np.fft.fftn(x)) <= 1e-12
        assert back.dtype == np.float64
        assert rel_inf(back, x) <= 1e-12


def _pfc_run(pkg, psi0, grid, steps, pg=None, G=1, real=True):
    from paper_2603_26818_b200 import distfft, pfc
    from paper_2603_26818_b200.pencil import pencil_scatter

    params = pfc.PfcParams()

    def body(w):
        sym = pkg.make_symbols(grid, -0.3)
        if pg is None:
            f = distfft.scatter(psi0, w, grid, distfft.Layout.Z_SLAB, real=real)
        else:
            f = pencil_scatter(psi0 if real else psi0.astype(np.complex128), w, grid, pg, real=real)
        st = pfc.PfcState(psi_hat=distfft.forward(f, w), grid=grid, symbols=sym, worker=w)
        e0 = pfc.free_energy(st, params)
        m0 = pfc.mean_and_max(st)
        pfc.pfc_run(st, params, steps)
        e1 = pfc.free_energy(st, params)
        m1 = pfc.mean_and_max(st)
        return distfft.gather(distfft.inverse(st.psi_hat, w), w), (e0, e1), (m0, m1)

    return pkg.spawn_group(G if pg is None else pg.size, body)[0]


@pytest.mark.parametrize("pr,pc", [(1, 2), (2, 1), (2, 2), (2, 4)])
@pytest.mark.parametrize("real", [True, False])
def test_pencil_pfc_equals_slab_bitwise(pkg, pr, pc, real):
    from paper_2603_26818_b200.pencil import PencilGrid
    from paper_2603_26818_b200.pfc import default_domain_length, initial_field

    n = (16, 16, 16)
    grid = pkg.GridSpec(n, default_domain_length(n))
    psi0 = initial_field("constant_plus_noise", grid, seed=4, noise_amplitude=0.05)
    slab, es, ms = _pfc_run(pkg, psi0, grid, 20, real=real)
    pen, ep, mp = _pfc_run(pkg, psi0, grid, 20, pg=PencilGrid(pr, pc), real=real)
    np.testing.assert_array_equal(pen, slab)
    assert ms[0][0] == mp[0][0] and ms[1][0] == mp[1][0]  # mean from the zero mode
    assert ep[1] == pytest.approx(es[1], rel=1e-12)


def test_pencil_pfc_32_vs_reference_golden(pkg, golden):
    from paper_2603_26818_b200.pencil import PencilGrid

    g = golden("pfc3d_32")
    grid = pkg.GridSpec((32, 32, 32), tuple(g["length"]))
    psi, e, m = _pfc_run(pkg, g["init"], grid, 100, pg=PencilGrid(2, 3))
    assert rel_l2(psi, g["psi"]) <= 1e-9
    assert e[1] == pytest.approx(g["energies"][-1], rel=1e-9)
