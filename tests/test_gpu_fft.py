"""CUDA parity of the serial and distributed transforms against the oracle
(numpy restatement of fftcore/distfft) and the reference's golden vectors.

Tolerance: relative max error <= 1e-12 per transform (north star), the
reference's own bar (test_acceptance.py:52-69)."""

import numpy as np
import pytest

from conftest import rel_inf, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_26818_b200 as p

    return p


def rand(shape, seed=0):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.mark.parametrize("n", list(range(1, 17)) + [31, 32, 64, 100, 128, 243, 256, 512, 750, 1000, 1024, 1400, 2048, 4096, 4099])
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_fft_axis_lengths(pkg, n, axis):
    import ref_numpy as ora

    shape = [3, 4, 5]
    shape[axis] = n
    if n >= 512:
        shape = [2, 3, 2]
        shape[axis] = n
    x = rand(tuple(shape), seed=n + 17 * axis)
    for fwd in (True, False):
        got = pkg.fft_axis(x, axis, forward=fwd)
        want = ora.fft_axis(x, axis, fwd)
        assert rel_inf(got, want) <= TOL, (n, axis, fwd, rel_inf(got, want))


def test_fft_against_reference_golden(pkg, golden):
    g = golden("fft_serial")
    i = 0
    while f"in{i}" in g:
        a = g[f"in{i}"]
        assert rel_inf(pkg.fft_nd(a), g[f"nd{i}"]) <= TOL
        assert rel_inf(pkg.fft_nd(a, forward=False), g[f"ind{i}"]) <= TOL
        for ax in range(3):
            assert rel_inf(pkg.fft_axis(a, ax), g[f"ax{i}_{ax}"]) <= TOL
        i += 1
    assert i >= 6


def test_brute_force_dft(pkg):
    import ref_numpy as ora

    x = rand((7, 5, 3), 3)
    assert rel_inf(pkg.fft_nd(x), ora.dft_nd(x)) <= TOL


def test_delta_constant_parseval(pkg):
    x = np.zeros((8, 8, 8), dtype=np.complex128)
    x[0, 0, 0] = 1.0
    np.testing.assert_array_equal(pkg.fft_nd(x), np.ones((8, 8, 8)))
    c = 2.5 - 0.5j
    out = pkg.fft_axis(np.full((16, 1, 1), c), 0)
    assert out[0, 0, 0] == 16 * c
    assert np.all(out[1:] == 0)
    y = rand((16, 32, 8), 5)
    Y = pkg.fft_nd(y)
    assert abs(np.sum(abs(y) ** 2) - np.sum(abs(Y) ** 2) / y.size) <= 1e-12 * np.sum(abs(y) ** 2)


def test_device_tensor_path(pkg):
    import torch

    x = rand((32, 16, 64), 9)
    t = torch.from_numpy(x).cuda()
    out = pkg.fft_nd(t)
    assert out.is_cuda
    assert rel_inf(out.cpu().numpy(), np.fft.fftn(x)) <= TOL
    back = pkg.fft_nd(out, forward=False)
    assert rel_inf(back.cpu().numpy(), x) <= TOL


def _dist(pkg, full, G, real=False):
    from paper_2603_26818_b200 import distfft

    grid = pkg.GridSpec(full.shape, (1.0, 1.0, 1.0))

    def body(w):
        f = distfft.scatter(full, w, grid, distfft.physical_layout(grid), real=real)
        spec = distfft.forward(f, w)
        back = distfft.inverse(spec, w)
        return distfft.gather(spec, w), distfft.gather(back, w), spec.local.shape

    return pkg.spawn_group(G, body)


@pytest.mark.parametrize("shape", [(4, 4, 4), (5, 5, 5), (6, 6, 6), (8, 8, 8), (12, 12, 12),
                                   (16, 16, 16), (8, 12, 16), (4, 4, 2), (32, 64, 16), (64, 64, 64)])
@pytest.mark.parametrize("G", [1, 2, 3, 4])
def test_distributed_c2c(pkg, shape, G):
    import ref_numpy as ora

    x = rand(shape, 11)
    res = _dist(pkg, x, G)
    want = ora.fft_nd(x)
    for spec, back, _ in res:
        assert rel_inf(spec, want) <= TOL
        assert rel_inf(back, x) <= TOL


@pytest.mark.parametrize("shape", [(8, 8, 1), (6, 9, 1), (256, 256, 1), (64, 32, 1)])
@pytest.mark.parametrize("G", [1, 2, 3])
def test_distributed_2d(pkg, shape, G):
    import ref_numpy as ora

    x = rand(shape, 12)
    spec, back, _ = _dist(pkg, x, G)[0]
    assert rel_inf(spec, ora.fft_nd(x)) <= TOL
    assert rel_inf(back, x) <= TOL


def test_distributed_golden(pkg, golden):
    g = golden("fft_dist")
    for i in range(3):
        spec, _, _ = _dist(pkg, g[f"in{i}"], 3)[0]
        assert rel_inf(spec, g[f"out{i}"]) <= TOL


@pytest.mark.parametrize("shape", [(4, 4, 4), (8, 8, 8), (16, 8, 4), (32, 32, 32), (64, 16, 8),
                                   (128, 128, 128), (8, 16, 1), (256, 256, 1)])
@pytest.mark.parametrize("G", [1, 2, 3, 4])
def test_distributed_r2c(pkg, shape, G):
    rng = np.random.default_rng(21)
    x = rng.standard_normal(shape)
    spec, back, local_shape = _dist(pkg, x, G, real=True)[0]
    want = np.fft.fftn(x)
    assert rel_inf(spec, want) <= TOL
    assert back.dtype == np.float64
    assert rel_inf(back, x) <= TOL
    # half spectrum: x modes split over the ranks
    assert sum(r[2][0] for r in _dist(pkg, x, G, real=True)) == shape[0] // 2 + 1


def test_r2c_kernels_direct(pkg):
    """rfft_x / irfft_x against numpy.fft.rfft along the slowest axis."""
    import torch
    from paper_2603_26818_b200 import _native as nat

    for nx in (4, 8, 16, 64, 256, 1024, 2048, 4096, 8192):
        inner = 3 if nx >= 4096 else 37
        x = np.random.default_rng(nx).standard_normal((nx, inner))
        t = torch.from_numpy(x).cuda()
        out = torch.empty((nx // 2 + 1, inner), dtype=torch.complex128, device="cuda")
        nat.call("pfcs_rfft_x", nat.ptr(t), nat.ptr(out), nx, inner, nat.stream_ptr())
        want = np.fft.rfft(x, axis=0)
        assert rel_inf(out.cpu().numpy(), want) <= TOL, nx
        back = torch.empty_like(t)
        nat.call("pfcs_irfft_x", nat.ptr(out), nat.ptr(back), nx, inner, nat.stream_ptr())
        assert rel_inf(back.cpu().numpy(), x) <= TOL, nx


def test_exchange_bookkeeping(pkg):
    """v(x,y,z) = 100x + 10y + z: after the transpose worker 1's local
    (0,2,3) is the global (2,2,3) entry (test_distfft.py:81-98)."""
    from paper_2603_26818_b200 import distfft

    grid = pkg.GridSpec((4, 4, 4), (1.0,) * 3)
    xs, ys, zs = np.meshgrid(*(np.arange(4),) * 3, indexing="ij")
    v = (100 * xs + 10 * ys + zs).astype(np.complex128)

    def body(w):
        out = distfft.exchange_z_to_x(distfft.scatter(v, w, grid, distfft.Layout.Z_SLAB), w)
        back = distfft.exchange_x_to_z(out, w)
        return out.local, back.local

    res = pkg.spawn_group(2, body)
    assert res[1][0][0, 2, 3] == 223
    np.testing.assert_array_equal(res[0][0], v[0:2])
    np.testing.assert_array_equal(res[1][1], v[:, :, 2:4])


def test_layout_errors(pkg):
    from paper_2603_26818_b200 import distfft

    grid = pkg.GridSpec((4, 4, 4), (1.0,) * 3)

    def body(w):
        f = distfft.scatter(rand((4, 4, 4)), w, grid, distfft.Layout.X_SLAB)
        distfft.exchange_z_to_x(f, w)

    with pytest.raises(Exception, match="expects Z_SLAB"):
        pkg.spawn_group(1, body)

    def body2(w):
        distfft.scatter(rand((4, 4, 5)), w, grid, distfft.Layout.Z_SLAB)

    with pytest.raises(Exception, match="does not match grid"):
        pkg.spawn_group(1, body2)


def test_large_roundtrip_512(pkg):
    """configs[1]: 512^3 R2C round trip on one GPU, relative L2 <= 1e-12."""
    import torch
    from paper_2603_26818_b200 import distfft

    n = 512
    grid = pkg.GridSpec((n, n, n), (1.0,) * 3)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((n, n, n), dtype=torch.float64, device="cuda", generator=g)

    def body(w):
        f = distfft.DistField(grid, distfft.Layout.Z_SLAB, distfft.Space.PHYSICAL, x)
        spec = distfft.forward(f, w)
        back = distfft.inverse(spec, w)
        # linearity/Parseval on the device: sum |x|^2 == sum |X|^2 / N (half-spectrum weights)
        return float(torch.linalg.vector_norm(back.dev - x) / torch.linalg.vector_norm(x))

    err = pkg.spawn_group(1, body)[0]
    assert err <= 1e-12


@pytest.mark.parametrize("shape", [(8, 8, 3), (6, 10, 4), (64, 32, 5), (256, 256, 1), (7, 12, 1)])
def test_fft_2d_vs_reference_order(pkg, shape):
    """fftcore.fft_2d (fftcore.py:43-45): axis 0 then axis 1 in both
    directions, every z-plane independently (oracle = the reference's own
    composition on pocketfft)."""
    import ref_numpy as ora

    x = rand(shape, 31)
    for fwd in (True, False):
        got = pkg.fft_2d(x, forward=fwd)
        want = ora.fft_2d(x, fwd)
        assert rel_inf(got, want) <= TOL
    # plane independence: each z plane is the 2D transform of that plane
    got = pkg.fft_2d(x)
    for z in range(shape[2]):
        assert rel_inf(got[:, :, z], np.fft.fft2(x[:, :, z])) <= TOL


@pytest.mark.parametrize("G", [1, 2, 3])
def test_exchange_2d_bookkeeping(pkg, G):
    """distfft.exchange_y_to_x / exchange_x_to_y (distfft.py:136-140) on a 2D
    grid: v(x, y) = 100 x + y; after Y->X each rank holds its x rows with
    all y, and X->Y restores the Y slab exactly (pure data movement)."""
    from paper_2603_26818_b200 import distfft
    from paper_2603_26818_b200.grid import slab_layout

    nx, ny = 7, 9
    grid = pkg.GridSpec((nx, ny, 1), (1.0,) * 3)
    xs, ys = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    v = (100 * xs + ys).astype(np.complex128)[:, :, None]

    def body(w):
        f = distfft.scatter(v, w, grid, distfft.Layout.Y_SLAB)
        out = distfft.exchange_y_to_x(f, w)
        back = distfft.exchange_x_to_y(out, w)
        return out.layout, out.local, back.layout, back.local, f.local

    xl = slab_layout(nx, G, axis=0)
    for r, (lay_out, out, lay_back, back, orig) in enumerate(pkg.spawn_group(G, body)):
        assert lay_out == distfft.Layout.X_SLAB and lay_back == distfft.Layout.Y_SLAB
        np.testing.assert_array_equal(out, v[xl.local_slice(r)])
        np.testing.assert_array_equal(back, orig)


def test_exchange_2d_layout_errors(pkg):
    from paper_2603_26818_b200 import distfft

    grid = pkg.GridSpec((4, 4, 1), (1.0,) * 3)

    def body(w):
        f = distfft.scatter(np.zeros((4, 4, 1), np.complex128), w, grid, distfft.Layout.X_SLAB)
        distfft.exchange_x_to_y(distfft.exchange_y_to_x(f, w), w)

    with pytest.raises(Exception, match="Y_SLAB"):
        pkg.spawn_group(1, body)
