"""Single-GPU plan C API (include/pfcs.h pfcs_plan_*): the whole hot path
from C, bit-identical to the Python path it mirrors (distfft.forward /
inverse and pfc.pfc_run at one rank)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_26818_b200 import _native

    return _native


def _plan(nat, nx, ny, nz):
    h = ctypes.c_void_p()
    nat.call("pfcs_plan_create", nx, ny, nz, ctypes.addressof(h))
    return h


@pytest.mark.parametrize("shape", [(32, 24, 16), (64, 8, 128), (16, 16, 16)])
def test_plan_matches_python_path(env, shape):
    import torch

    from paper_2603_26818_b200 import distfft, pfc
    from paper_2603_26818_b200.distfft import DistField, Layout, Space
    from paper_2603_26818_b200.grid import GridSpec, make_symbols
    from paper_2603_26818_b200.transport import Worker, WorkerGroup

    nat = env
    dev = torch.device("cuda", 0)
    w = Worker(WorkerGroup(1), 0, dev)
    grid = GridSpec(shape, pfc.default_domain_length(shape))
    nx, ny, nz = shape
    nh = nx // 2 + 1
    gen = torch.Generator(device=dev).manual_seed(5)
    x = (-0.3 + 0.02 * (torch.rand(shape, dtype=torch.float64, device=dev, generator=gen) - 0.5)).contiguous()
    h = _plan(nat, nx, ny, nz)
    try:
        assert nat.load().pfcs_plan_spectral_elems(h) == nh * ny * nz
        st = nat.stream_ptr()
        spec_c = torch.empty(nh * ny * nz, dtype=torch.complex128, device=dev)
        nat.call("pfcs_plan_fwd", h, nat.ptr(x), nat.ptr(spec_c), st)
        spec_py = distfft.forward(DistField(grid, Layout.Z_SLAB, Space.PHYSICAL, x), w)
        assert torch.equal(spec_c, spec_py.dev.reshape(-1))
        back_c = torch.empty_like(x)
        work = torch.empty_like(spec_c)
        nat.call("pfcs_plan_inv", h, nat.ptr(spec_c), nat.ptr(back_c), nat.ptr(work), st)
        assert torch.equal(back_c.reshape(-1), distfft.inverse(spec_py, w).dev.reshape(-1))

        hl = distfft._layout(grid, Layout.X_SLAB, 1, True)
        sym = make_symbols(grid, -0.3, layout=hl, rank=0)
        state = pfc.PfcState(psi_hat=spec_py, grid=grid, symbols=sym, worker=w)
        psi_c = spec_c.clone()
        pfc.pfc_run(state, pfc.PfcParams(), 7)
        eng = pfc._engine(state)
        kx, ky, kz = pfc.slab_kvectors(grid, sym, eng.g, dev)
        diag = torch.empty(7 * nat.DIAG_SLOTS * nat.DIAG_VALS, dtype=torch.float64, device=dev)
        nat.call("pfcs_plan_pfc_steps", h, nat.ptr(psi_c), nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), -0.3, 0.1, 7,
                 nat.ptr(diag), nat.ptr(work), st)
        torch.cuda.synchronize()
        assert torch.equal(psi_c, state.psi_hat.dev.reshape(-1))
        assert np.isfinite(diag.cpu().numpy()).all()
    finally:
        nat.call("pfcs_plan_destroy", h)


def test_plan_rejects_unsupported(env):
    nat = env
    h = ctypes.c_void_p()
    with pytest.raises(Exception):
        nat.call("pfcs_plan_create", 24, 8, 8, ctypes.addressof(h))  # nx not a power of two
    with pytest.raises(Exception):
        nat.call("pfcs_plan_create", 32, 8, 12, ctypes.addressof(h))  # nz not a power of two
