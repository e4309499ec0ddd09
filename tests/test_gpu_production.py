"""Parity at the sizes the bench times (VERDICT r1 "pin parity at the sizes you
benchmark").

The small-grid tests elsewhere take the narrow-tile fallback of the kernels
(fewer tiles than SMs); here every (kernel, line length) that bench.py
launches runs with inner extents large enough for the DEFAULT production
tile (and several tiles per persistent CTA, so the TMA / register pipelines
alternate stages), and is compared with numpy/scipy pocketfft — the
reference's own FFT (fftcore.py:31-40) — at the per-transform bar of the
reference's acceptance test (test_acceptance.py:52-69, relative L2 <= 1e-12).

Then the benchmarked workloads themselves:
  * configs[1] 512^3: forward R2C and C2C spectra vs scipy rfftn / fftn and
    inverse of the scipy spectrum (not only the round trip);
  * 512^3 PFC, 10 steps vs the lean R2C restatement of pfc.py:96-128
    (oracle/ref_numpy.py:pfc_step_r2c_lean), field <= 1e-9;
  * 1024^3 PFC (configs[2] grid): G = 1 bit-identical to G = 2, 3 and 4 (thread
    ranks on one GPU: blocked z kernels, fused peer-scatter kernels at the
    production tiles), and 1 step vs the lean restatement when the host has
    the RAM for it.
"""

import os

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

WORKERS = os.cpu_count() or 1
TOL = 1e-12


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    return torch


def _nat():
    from paper_2603_26818_b200 import _native as nat

    return nat


def _cplx(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _to(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ------------------------------------------------------------- line kernels --

# (outer, n, inner): TMA y pass at 512 (T = 8) and 1024 (T = 4); the 2048-point
# register-loaded y pass (T = 4).  >= 3 tiles per persistent CTA.
STRIDED = [(3, 512, 1200), (2, 1024, 1500), (2, 2048, 700)]


@pytest.mark.parametrize("outer,n,inner", STRIDED)
@pytest.mark.parametrize("fwd", [1, 0])
def test_strided_pass_production_tiles(torch_cuda, outer, n, inner, fwd):
    import scipy.fft as sfft

    torch, nat = torch_cuda, _nat()
    x = _cplx(np.random.default_rng(n + inner + fwd), (outer, n, inner))
    a = _to(torch, x)
    b = torch.empty_like(a)
    nat.call("pfcs_fft_axis_c2c", nat.ptr(a), nat.ptr(b), outer, n, inner, 1, fwd, nat.stream_ptr())
    want = sfft.fft(x, axis=1, workers=WORKERS) if fwd else sfft.ifft(x, axis=1, workers=WORKERS)
    assert rel_l2(b.cpu().numpy(), want) <= TOL
    # in place (the PFC step's y passes)
    nat.call("pfcs_fft_axis_c2c", nat.ptr(a), nat.ptr(a), outer, n, inner, 1, fwd, nat.stream_ptr())
    assert torch.equal(a, b)


# contiguous z lines (k_lines at 512: T = 1, 2-stage register pipeline;
# 1024 / 2048: T = 1), many more lines than resident CTAs
ZLINES = [(20, 300, 512), (10, 500, 1024), (5, 500, 2048)]


@pytest.mark.parametrize("n0,n1,nz", ZLINES)
@pytest.mark.parametrize("fwd", [1, 0])
def test_zlines_production_tiles(torch_cuda, n0, n1, nz, fwd):
    import scipy.fft as sfft

    torch, nat = torch_cuda, _nat()
    x = _cplx(np.random.default_rng(nz + fwd), (n0, n1, nz))
    a = _to(torch, x)
    b = torch.empty_like(a)
    nat.call("pfcs_fft_axis_c2c", nat.ptr(a), nat.ptr(b), n0, n1, nz, 2, fwd, nat.stream_ptr())
    want = sfft.fft(x, axis=2, workers=WORKERS) if fwd else sfft.ifft(x, axis=2, workers=WORKERS)
    assert rel_l2(b.cpu().numpy(), want) <= TOL


def _blocked(a, G):
    """(nlines, nz) -> the blocked layout of distfft._exchange's receive
    buffer: z slab g stored densely as (nlines, cz_g), slabs concatenated."""
    from ref_numpy import slab_counts

    offs = np.concatenate([[0], np.cumsum(slab_counts(a.shape[1], G))])
    return np.concatenate([a[:, offs[g]:offs[g + 1]].ravel() for g in range(G)])


@pytest.mark.parametrize("nz", [512, 1024, 2048])
@pytest.mark.parametrize("g_in,g_out", [(1, 4), (4, 1), (3, 8)])
def test_zlines_blocked_production(torch_cuda, nz, g_in, g_out):
    """pfcs_fft_zlines with blocked input/output (the slab pipeline's
    transposes, distfft.py:110-124) at the G > 1 production line lengths."""
    import scipy.fft as sfft

    torch, nat = torch_cuda, _nat()
    nlines = 2400 if nz <= 1024 else 1200
    x = _cplx(np.random.default_rng(nz * g_in + g_out), (nlines, nz))
    fwd = 1 if g_in > 1 else 0
    a = _to(torch, _blocked(x, g_in))
    b = torch.empty_like(a)
    nat.call("pfcs_fft_zlines", nat.ptr(a), nat.ptr(b), nlines, nz, g_in, g_out, fwd, nat.stream_ptr())
    want = sfft.fft(x, axis=1, workers=WORKERS) if fwd else sfft.ifft(x, axis=1, workers=WORKERS)
    assert rel_l2(b.cpu().numpy(), _blocked(want, g_out)) <= TOL


# x passes: R2C / C2R / fused cube at nx = 512 (16-line TMA tiles), 1024
# (8-line tiles; R2C register pipeline, C2R and cube TMA), 2048 (4-line
# tiles); inner >= 3 tiles per CTA at one CTA per SM
XCASES = [(512, 7104), (1024, 3600), (2048, 2400)]


@pytest.mark.parametrize("nx,inner", XCASES)
def test_real_x_production_tiles(torch_cuda, nx, inner):
    import scipy.fft as sfft

    torch, nat = torch_cuda, _nat()
    rng = np.random.default_rng(nx)
    r = rng.standard_normal((nx, inner))
    h = torch.empty((nx // 2 + 1, inner), dtype=torch.complex128, device="cuda")
    nat.call("pfcs_rfft_x", nat.ptr(_to(torch, r)), nat.ptr(h), nx, inner, nat.stream_ptr())
    want = sfft.rfft(r, axis=0, workers=WORKERS)
    assert rel_l2(h.cpu().numpy(), want) <= TOL
    # C2R of a spectrum with the DC / Nyquist imaginary parts set (ignored,
    # numpy irfft convention)
    spec = _cplx(rng, (nx // 2 + 1, inner))
    out = torch.empty((nx, inner), dtype=torch.float64, device="cuda")
    nat.call("pfcs_irfft_x", nat.ptr(_to(torch, spec)), nat.ptr(out), nx, inner, nat.stream_ptr())
    assert rel_l2(out.cpu().numpy(), sfft.irfft(spec, n=nx, axis=0, workers=WORKERS)) <= TOL


@pytest.mark.parametrize("nx,inner", XCASES)
def test_cube_x_production_tiles(torch_cuda, nx, inner):
    """pfcs_pfc_cube_x (C2R -> x*x*x -> R2C, pfc.py:109 fused into the x
    stage) vs irfft -> cube -> rfft, with its max|psi| diagnostic."""
    import scipy.fft as sfft

    torch, nat = torch_cuda, _nat()
    rng = np.random.default_rng(nx + 1)
    psi = -0.3 + 0.1 * rng.standard_normal((nx, inner))
    spec = sfft.rfft(psi, axis=0, workers=WORKERS)
    d = _to(torch, spec)
    diag = torch.zeros(nat.DIAG_SLOTS * nat.DIAG_VALS, dtype=torch.float64, device="cuda")
    nat.call("pfcs_pfc_cube_x", nat.ptr(d), nx, inner, 1, nat.ptr(diag), nat.stream_ptr())
    phys = sfft.irfft(spec, n=nx, axis=0, workers=WORKERS)
    want = sfft.rfft(phys * phys * phys, axis=0, workers=WORKERS)
    assert rel_l2(d.cpu().numpy(), want) <= TOL
    dg = diag.cpu().numpy().reshape(nat.DIAG_SLOTS, nat.DIAG_VALS)
    assert abs(dg[:, 2].max() - np.abs(phys).max()) <= 1e-13 * np.abs(phys).max()
    assert dg[:, 3].max() == 0


# fused z update + next inverse (k_pfc_z) at nz = 512 / 1024 / 2048
ZUPD = [(8, 600, 512), (4, 600, 1024), (2, 600, 2048)]


@pytest.mark.parametrize("cx,ny,nz", ZUPD)
def test_pfc_update_z_production(torch_cuda, cx, ny, nz):
    """pfcs_pfc_update_z: forward z FFT of N, the implicit update
    (pfc.py:114-121, symbols of grid.py:155-208 from the 1D k vectors) and
    the inverse z FFT of the new psi_hat."""
    import scipy.fft as sfft

    from ref_numpy import wavenumbers

    torch, nat = torch_cuda, _nat()
    rng = np.random.default_rng(nz)
    nl = _cplx(rng, (cx, ny, nz))
    psi = _cplx(rng, (cx, ny, nz))
    L = 2 * np.pi * np.sqrt(3) * 8
    kx = wavenumbers(2 * cx, L)[:cx]
    ky = wavenumbers(ny, L)
    kz = wavenumbers(nz, L)
    eps, dt = -0.3, 0.1
    k2 = (kx[:, None, None] ** 2 + ky[None, :, None] ** 2) + kz[None, None, :] ** 2
    lap = -k2
    lin = lap * (eps + ((1.0 - k2) * (1.0 - k2)) * ((4.0 / 3.0 - k2) * (4.0 / 3.0 - k2)))
    new = (psi + dt * (lap * sfft.fft(nl, axis=2, workers=WORKERS))) / (1.0 - dt * lin)
    nxt = sfft.ifft(new, axis=2, workers=WORKERS)
    a, p = _to(torch, nl), _to(torch, psi)
    o = torch.empty_like(a)
    diag = torch.zeros(nat.DIAG_SLOTS * nat.DIAG_VALS, dtype=torch.float64, device="cuda")
    kd = [_to(torch, v) for v in (kx, ky, kz)]
    nat.call("pfcs_pfc_update_z", nat.ptr(a), nat.ptr(p), nat.ptr(o), cx, ny, nz, 1, 1,
             *(nat.ptr(v) for v in kd), eps, dt, nat.ptr(diag), nat.stream_ptr())
    assert rel_l2(p.cpu().numpy(), new) <= TOL
    assert rel_l2(o.cpu().numpy(), nxt) <= TOL
    assert diag.cpu().numpy().reshape(nat.DIAG_SLOTS, nat.DIAG_VALS)[:, 3].max() == 0


# ------------------------------------------------- configs[1]: 512^3 spectra --

def _world1():
    from paper_2603_26818_b200.transport import Worker, WorkerGroup

    import torch

    return Worker(WorkerGroup(1), 0, torch.device("cuda", 0))


@pytest.mark.parametrize("kind", ["r2c", "c2c"])
def test_512_forward_inverse_vs_pocketfft(torch_cuda, kind):
    """configs[1]: the 512^3 forward spectrum (distfft.forward, distfft.py:
    150-160) vs pocketfft's 3D transform, and the inverse of pocketfft's
    spectrum (distfft.py:163-173) vs the field: relative L2 <= 1e-12 each."""
    import scipy.fft as sfft

    import paper_2603_26818_b200 as pkg
    from paper_2603_26818_b200 import distfft

    torch = torch_cuda
    n = 512
    grid = pkg.GridSpec((n, n, n), (1.0,) * 3)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((n, n, n))
    if kind == "c2c":
        x = x + 1j * rng.standard_normal((n, n, n))
    w = _world1()
    f = distfft.DistField(grid, distfft.Layout.Z_SLAB, distfft.Space.PHYSICAL, _to(torch, x))
    spec = distfft.forward(f, w)
    got = spec.dev.cpu().numpy()
    del spec, f
    if kind == "r2c":
        want = sfft.rfftn(x, axes=(1, 2, 0), workers=WORKERS)  # x halved (axis 0 last)
    else:
        want = sfft.fftn(x, workers=WORKERS)
    assert got.shape == want.shape
    assert rel_l2(got, want) <= TOL
    del got
    sp = distfft.DistField(grid, distfft.Layout.X_SLAB, distfft.Space.SPECTRAL, _to(torch, want),
                           half=(kind == "r2c"))
    back = distfft.inverse(sp, w).dev.cpu().numpy()
    assert rel_l2(back, x) <= TOL
    torch.cuda.empty_cache()


# ------------------------------------------------------ PFC at bench sizes --

def _pfc_state(pkg, w, grid, x_dev):
    from paper_2603_26818_b200 import distfft, pfc

    lay = distfft._layout(grid, distfft.Layout.X_SLAB, w.size, True)
    sym = pkg.make_symbols(grid, -0.3, layout=lay, rank=w.rank)
    f = distfft.DistField(grid, distfft.Layout.Z_SLAB, distfft.Space.PHYSICAL, x_dev)
    return pfc.PfcState(psi_hat=distfft.forward(f, w), grid=grid, symbols=sym, worker=w)


def _host_gib() -> float:
    try:
        import psutil

        return psutil.virtual_memory().available / 2**30
    except Exception:
        return 0.0


def test_pfc_512_10_steps_vs_lean_restatement(torch_cuda):
    """512^3 PFC, 10 fused steps vs oracle.pfc_step_r2c_lean (pocketfft,
    pfc.py:96-128 arithmetic), relative L2 <= 1e-9 (north star) on psi_hat;
    mean mode bit-invariant."""
    import ref_numpy as ora

    import paper_2603_26818_b200 as pkg
    from paper_2603_26818_b200 import pfc

    if _host_gib() < 24:
        pytest.skip("host RAM < 24 GiB for the 512^3 restatement")
    torch = torch_cuda
    n = (512,) * 3
    grid = pkg.GridSpec(n, pfc.default_domain_length(n))
    x = -0.3 + np.random.default_rng(5).uniform(-0.01, 0.01, n)
    w = _world1()
    st = _pfc_state(pkg, w, grid, _to(torch, x))
    want = st.psi_hat.dev.cpu().numpy()
    mean0 = want[0, 0, 0].real
    pfc.pfc_run(st, pfc.PfcParams(), 10)
    got = st.psi_hat.dev.cpu().numpy()
    for _ in range(10):
        want = ora.pfc_step_r2c_lean(want, n, grid.length, -0.3, 0.1, workers=WORKERS)
    assert rel_l2(got, want) <= 1e-9
    assert got[0, 0, 0].real == mean0
    del st
    torch.cuda.empty_cache()


@pytest.fixture(scope="module")
def pfc1024(torch_cuda):
    """1024^3 (configs[2] grid) G = 1 reference run on one GPU: the initial
    field (device), psi_hat after 3 fused steps."""
    import paper_2603_26818_b200 as pkg
    from paper_2603_26818_b200 import pfc

    torch = torch_cuda
    n = (1024,) * 3
    grid = pkg.GridSpec(n, pfc.default_domain_length(n))
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g).mul_(0.02).add_(-0.31)
    st = _pfc_state(pkg, _world1(), grid, x)
    spec0 = st.psi_hat.dev.clone()
    pfc.pfc_run(st, pfc.PfcParams(), 3)
    out = {"grid": grid, "x": x, "spec0": spec0, "psi_hat3": st.psi_hat.dev}
    del st
    yield out
    out.clear()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("G", [2, 3, 4])
def test_pfc_1024_G_invariance(torch_cuda, pfc1024, G):
    """1024^3, 3 steps: G thread ranks (slab decomposition, fused peer
    exchange, blocked z kernels at production tiles; G = 3 splits both the
    513 x modes and the 1024 z planes unevenly) reproduce the G = 1 spectrum
    bit for bit (reference property, README.md:5-7)."""
    import paper_2603_26818_b200 as pkg
    from paper_2603_26818_b200 import pfc
    from paper_2603_26818_b200.grid import slab_layout

    torch = torch_cuda
    grid, x = pfc1024["grid"], pfc1024["x"]
    zl = slab_layout(1024, G)
    xl = slab_layout(513, G)

    def body(w):
        z0 = zl.offsets[w.rank]
        slab = x[:, :, z0:z0 + zl.counts[w.rank]].contiguous()
        st = _pfc_state(pkg, w, grid, slab)
        pfc.pfc_run(st, pfc.PfcParams(), 3)
        x0 = xl.offsets[w.rank]
        ok = torch.equal(st.psi_hat.dev, pfc1024["psi_hat3"][x0:x0 + xl.counts[w.rank]])
        del st
        return ok

    assert all(pkg.spawn_group(G, body))
    torch.cuda.empty_cache()


def test_pfc_1024_step_vs_lean_restatement(torch_cuda, pfc1024):
    """1024^3: one fused step vs the lean R2C restatement on the box host
    (needs ~60 GiB of host RAM; skipped otherwise)."""
    import ref_numpy as ora

    import paper_2603_26818_b200 as pkg
    from paper_2603_26818_b200 import pfc

    if _host_gib() < 80:
        pytest.skip("host RAM < 80 GiB for the 1024^3 restatement")
    torch = torch_cuda
    grid = pfc1024["grid"]
    spec0 = pfc1024["spec0"]
    w = _world1()
    from paper_2603_26818_b200 import distfft

    lay = distfft._layout(grid, distfft.Layout.X_SLAB, 1, True)
    st = pfc.PfcState(psi_hat=distfft.DistField(grid, distfft.Layout.X_SLAB, distfft.Space.SPECTRAL,
                                                spec0.clone(), half=True),
                      grid=grid, symbols=pkg.make_symbols(grid, -0.3, layout=lay), worker=w)
    pfc.pfc_step(st, pfc.PfcParams())
    got = st.psi_hat.dev.cpu().numpy()
    del st
    torch.cuda.empty_cache()
    want = ora.pfc_step_r2c_lean(spec0.cpu().numpy(), grid.n, grid.length, -0.3, 0.1, workers=WORKERS)
    assert rel_l2(got, want) <= 1e-12


@pytest.mark.parametrize("nx,inner", [(512, 7104), (512, 7110), (1024, 3600), (1024, 3606), (64, 300)])
@pytest.mark.parametrize("kind", [0, 1, 3])
def test_rfft_x_prologue_production(torch_cuda, nx, inner, kind):
    """pfcs_rfft_x_pro (the R2C multiphysics transforms' fused psi^3, psi*g,
    alpha (c^3 - c)) at the production tiles (TMA path at nx 512, register
    path at 1024, small-tile fallback at 64): bit-identical to
    pfcs_real_pointwise followed by pfcs_rfft_x, and vs scipy <= 1e-12."""
    import scipy.fft as sfft

    torch, nat = torch_cuda, _nat()
    rng = np.random.default_rng(nx + kind)
    x = -0.3 + 0.2 * rng.standard_normal((nx, inner))
    g = rng.standard_normal((nx, inner))
    xd, gd = _to(torch, x), _to(torch, g)
    st = nat.stream_ptr()
    fused = torch.empty((nx // 2 + 1, inner), dtype=torch.complex128, device="cuda")
    nat.call("pfcs_rfft_x_pro", nat.ptr(xd), nat.ptr(fused), nx, inner, kind, nat.ptr(gd) if kind == 1 else None,
             0.7, st)
    pw = torch.empty_like(xd)
    nat.call("pfcs_real_pointwise", kind, nat.ptr(xd), nat.ptr(gd) if kind == 1 else None, None, None, None, None,
             nat.ptr(pw), pw.numel(), 0.7, st)
    two = torch.empty_like(fused)
    nat.call("pfcs_rfft_x", nat.ptr(pw), nat.ptr(two), nx, inner, st)
    assert torch.equal(fused, two)
    f = {0: x * x * x, 1: x * g, 3: 0.7 * (x * (x * x) - x)}[kind]
    assert rel_l2(fused.cpu().numpy(), sfft.rfft(f, axis=0, workers=WORKERS)) <= TOL


@pytest.mark.parametrize("nx,inner", [(512, 7104), (512, 7110), (1024, 3600), (64, 300)])
def test_xmul_x_production(torch_cuda, nx, inner):
    """pfcs_xmul_x (the x pass of the force product: C2R, times a real
    field, R2C, in place) at the production tiles: bit-identical to
    pfcs_irfft_x + pfcs_real_pointwise kind 1 + pfcs_rfft_x, and vs scipy
    <= 1e-12."""
    import scipy.fft as sfft

    torch, nat = torch_cuda, _nat()
    rng = np.random.default_rng(nx + inner)
    nh = nx // 2 + 1
    spec = rng.standard_normal((nh, inner)) + 1j * rng.standard_normal((nh, inner))
    g = rng.standard_normal((nx, inner))
    gd = _to(torch, g)
    st = nat.stream_ptr()
    fused = _to(torch, spec)
    nat.call("pfcs_xmul_x", nat.ptr(fused), nat.ptr(gd), nx, inner, st)
    phys = torch.empty((nx, inner), dtype=torch.float64, device="cuda")
    nat.call("pfcs_irfft_x", nat.ptr(_to(torch, spec)), nat.ptr(phys), nx, inner, st)
    prod = torch.empty_like(phys)
    nat.call("pfcs_real_pointwise", 1, nat.ptr(phys), nat.ptr(gd), None, None, None, None, nat.ptr(prod),
             prod.numel(), 0.0, st)
    two = torch.empty_like(fused)
    nat.call("pfcs_rfft_x", nat.ptr(prod), nat.ptr(two), nx, inner, st)
    assert torch.equal(fused, two)
    want = sfft.rfft(sfft.irfft(spec, n=nx, axis=0, workers=WORKERS) * g, axis=0, workers=WORKERS)
    assert rel_l2(fused.cpu().numpy(), want) <= TOL


@pytest.mark.parametrize("nx,inner", [(512, 7104), (512, 7110), (256, 3000), (256, 40)])
@pytest.mark.parametrize("with_dx", [False, True])
def test_xdot3_x_production(torch_cuda, nx, inner, with_dx):
    """pfcs_xdot3_x (the advection x pass: three C2R, (v0 g0 + v1 g1) + v2 g2,
    R2C) at production and small tiles: bit-identical to three
    pfcs_irfft_x + pfcs_real_pointwise kind 2 + pfcs_rfft_x (with dx: after
    pfcs_mul_deriv(axis 0) on the first spectrum), and vs scipy <= 1e-12;
    nx without the fused kernel is reported, not run."""
    import scipy.fft as sfft

    torch, nat = torch_cuda, _nat()
    assert nat.load().pfcs_xdot3_supported(nx, inner) == 1
    assert nat.load().pfcs_xdot3_supported(1024, inner) == 0
    rng = np.random.default_rng(nx * 3 + inner + with_dx)
    nh = nx // 2 + 1
    spec = rng.standard_normal((3, nh, inner)) + 1j * rng.standard_normal((3, nh, inner))
    vel = [rng.standard_normal((nx, inner)) for _ in range(3)]
    dxv = rng.standard_normal(nh)
    vd = [_to(torch, x) for x in vel]
    dxd = _to(torch, dxv)
    st = nat.stream_ptr()
    sd = [_to(torch, spec[a]) for a in range(3)]
    fused = torch.empty((nh, inner), dtype=torch.complex128, device="cuda")
    nat.call("pfcs_xdot3_x", nat.ptr(sd[0]), nat.ptr(sd[1]), nat.ptr(sd[2]), nat.ptr(vd[0]), nat.ptr(vd[1]),
             nat.ptr(vd[2]), nat.ptr(fused), nx, inner, nat.ptr(dxd) if with_dx else None, st)
    s0 = sd[0].clone()
    if with_dx:
        nat.call("pfcs_mul_deriv", nat.ptr(s0), nat.ptr(s0), nh, inner, 1, nat.ptr(dxd), 0, st)
    g = []
    for a, sa in enumerate([s0, sd[1], sd[2]]):
        ga = torch.empty((nx, inner), dtype=torch.float64, device="cuda")
        nat.call("pfcs_irfft_x", nat.ptr(sa), nat.ptr(ga), nx, inner, st)
        g.append(ga)
    prod = torch.empty_like(g[0])
    nat.call("pfcs_real_pointwise", 2, nat.ptr(vd[0]), nat.ptr(g[0]), nat.ptr(vd[1]), nat.ptr(g[1]), nat.ptr(vd[2]),
             nat.ptr(g[2]), nat.ptr(prod), prod.numel(), 0.0, st)
    two = torch.empty_like(fused)
    nat.call("pfcs_rfft_x", nat.ptr(prod), nat.ptr(two), nx, inner, st)
    assert torch.equal(fused, two)
    s0h = spec[0] * (1j * dxv[:, None]) if with_dx else spec[0]
    phys = [sfft.irfft(x, n=nx, axis=0, workers=WORKERS) for x in (s0h, spec[1], spec[2])]
    want = sfft.rfft((vel[0] * phys[0] + vel[1] * phys[1]) + vel[2] * phys[2], axis=0, workers=WORKERS)
    assert rel_l2(fused.cpu().numpy(), want) <= TOL
    with pytest.raises(Exception):
        nat.call("pfcs_xdot3_x", nat.ptr(sd[0]), nat.ptr(sd[1]), nat.ptr(sd[2]), nat.ptr(vd[0]), nat.ptr(vd[1]),
                 nat.ptr(vd[2]), nat.ptr(fused), 1024, inner // 2, None, st)

@pytest.mark.parametrize("shape", [(257, 64, 512), (9, 12, 1024), (5, 6, 12)])
def test_hydro_mu_z(torch_cuda, shape):
    """pfcs_hydro_mu_z (mu_hat with its operands' forward z passes fused) ==
    two forward z passes + pfcs_hydro_mu, bit for bit (fused kernel on
    power-of-two z; the two-pass form otherwise)."""
    torch, nat = torch_cuda, _nat()
    rng = np.random.default_rng(sum(shape))
    n0, n1, n2 = shape
    nl = _to(torch, rng.standard_normal(shape) + 1j * rng.standard_normal(shape))
    f = _to(torch, rng.standard_normal(shape) + 1j * rng.standard_normal(shape))
    kx, ky, kz = (_to(torch, rng.standard_normal(m)) for m in shape)
    st = nat.stream_ptr()
    mu = torch.empty_like(nl)
    nl_in, f_in = nl.clone(), f.clone()  # (the two-pass fallback transforms its operands in place)
    nl_out = torch.empty_like(nl)
    nat.call("pfcs_hydro_mu_z", nat.ptr(nl_in), nat.ptr(f_in), nat.ptr(mu), nat.ptr(nl_out), n0, n1, n2,
             nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), -0.3, st)
    a, b = nl.clone(), f.clone()
    nat.call("pfcs_fft_axis_c2c", nat.ptr(a), nat.ptr(a), n0, n1, n2, 2, 1, st)
    nat.call("pfcs_fft_axis_c2c", nat.ptr(b), nat.ptr(b), n0, n1, n2, 2, 1, st)
    want = torch.empty_like(nl)
    nat.call("pfcs_hydro_mu", nat.ptr(a), nat.ptr(b), nat.ptr(want), n0, n1, n2, nat.ptr(kx), nat.ptr(ky),
             nat.ptr(kz), -0.3, st)
    torch.cuda.synchronize()
    assert torch.equal(mu, want)
    assert torch.equal(nl_out, a)  # the finished F(psi^3) the next step reuses


@pytest.mark.parametrize("shape", [(257, 64, 512), (9, 12, 1024), (5, 6, 16)])
def test_hydro_mu_zgrad(torch_cuda, shape):
    """pfcs_hydro_mu_zgrad (mu_hat with grad mu's first inverse z passes:
    plain and with i k_z) == pfcs_hydro_mu_z + pfcs_fft_axis_c2c (inverse z)
    + pfcs_fft_axis_c2c_pro (inverse z, derivative prologue), bit for bit."""
    torch, nat = torch_cuda, _nat()
    rng = np.random.default_rng(3 + sum(shape))
    n0, n1, n2 = shape
    nl = _to(torch, rng.standard_normal(shape) + 1j * rng.standard_normal(shape))
    f = _to(torch, rng.standard_normal(shape) + 1j * rng.standard_normal(shape))
    kx, ky, kz, dz = (_to(torch, rng.standard_normal(m)) for m in (n0, n1, n2, n2))
    st = nat.stream_ptr()
    mu, nlo = torch.empty_like(nl), torch.empty_like(nl)
    nat.call("pfcs_hydro_mu_z", nat.ptr(nl), nat.ptr(f), nat.ptr(mu), nat.ptr(nlo), n0, n1, n2, nat.ptr(kx),
             nat.ptr(ky), nat.ptr(kz), -0.3, st)
    t0_w, tz_w = torch.empty_like(nl), torch.empty_like(nl)
    nat.call("pfcs_fft_axis_c2c", nat.ptr(mu), nat.ptr(t0_w), n0, n1, n2, 2, 0, st)
    nat.call("pfcs_fft_axis_c2c_pro", nat.ptr(mu), nat.ptr(tz_w), n0, n1, n2, 2, 0, 3, nat.ptr(dz), 2, st)
    t0, tz, nlo2 = torch.empty_like(nl), torch.empty_like(nl), torch.empty_like(nl)
    nat.call("pfcs_hydro_mu_zgrad", nat.ptr(nl), nat.ptr(f), None, nat.ptr(nlo2), nat.ptr(t0), nat.ptr(tz), nat.ptr(dz),
             n0, n1, n2, nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), -0.3, st)
    torch.cuda.synchronize()
    assert torch.equal(t0, t0_w) and torch.equal(tz, tz_w) and torch.equal(nlo2, nlo)
