"""Fused pointwise prologues (pfcs_fft_axis_c2c_pro) are bit-identical to the
standalone pointwise kernel followed by the plain pass, for every prologue,
axis and direction, on power-of-two (fused kernels) and other (two-kernel
fallback) lengths."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nat():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_26818_b200 import _native

    return _native


@pytest.mark.parametrize("shape", [(16, 8, 32), (32, 12, 64), (12, 10, 9), (64, 4, 4)])
@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("fwd", [1, 0])
def test_prologue_bit_identical(nat, shape, axis, fwd):
    import torch

    rng = np.random.default_rng(sum(shape) + axis)
    C = torch.complex128
    x = torch.from_numpy(rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).cuda()
    a = torch.from_numpy(rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).cuda()
    st = nat.stream_ptr()
    n0, n1, n2 = shape
    for pro in (1, 2, 3):
        for aux_axis in ((0, 1, 2) if pro == 3 else (0,)):
            d = torch.from_numpy(rng.standard_normal(shape[aux_axis])).cuda()
            aux = a if pro == 2 else (d if pro == 3 else None)
            want = torch.empty_like(x)
            if pro == 1:
                want.copy_(x)
                nat.call("pfcs_pfc_cube", nat.ptr(want), want.numel(), 0, None, st)
            elif pro == 2:
                nat.call("pfcs_cmul", nat.ptr(a), nat.ptr(x), nat.ptr(want), x.numel(), st)
            else:
                nat.call("pfcs_mul_deriv", nat.ptr(x), nat.ptr(want), n0, n1, n2, nat.ptr(d), aux_axis, st)
            nat.call("pfcs_fft_axis_c2c", nat.ptr(want), nat.ptr(want), n0, n1, n2, axis, fwd, st)
            got = torch.empty_like(x)
            nat.call("pfcs_fft_axis_c2c_pro", nat.ptr(x), nat.ptr(got), n0, n1, n2, axis, fwd, pro,
                     nat.ptr(aux) if aux is not None else None, aux_axis, st)
            torch.cuda.synchronize()
            assert torch.equal(got, want), (pro, aux_axis)
    del C


def test_prologue_argument_errors(nat):
    import torch

    x = torch.zeros((4, 4, 4), dtype=torch.complex128, device="cuda")
    with pytest.raises(Exception):
        nat.call("pfcs_fft_axis_c2c_pro", nat.ptr(x), nat.ptr(x), 4, 4, 4, 0, 1, 9, None, 0, nat.stream_ptr())
    with pytest.raises(Exception):
        nat.call("pfcs_fft_axis_c2c_pro", nat.ptr(x), nat.ptr(x), 4, 4, 4, 0, 1, 2, None, 0, nat.stream_ptr())
    with pytest.raises(Exception):
        nat.call("pfcs_fft_axis_c2c_pro", nat.ptr(x), nat.ptr(x), 4, 4, 4, 0, 1, 2, nat.ptr(x), 0, nat.stream_ptr())


@pytest.mark.parametrize("shape", [(9, 16, 512), (5, 12, 64), (6, 10, 9), (3, 4, 1), (33, 8, 2)])
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_update_zinv_bit_identical(nat, shape, kind):
    """pfcs_update_zinv (a spectral update fused into the z pass of the
    following inverse) ≡ the standalone update kernel + pfcs_fft_axis_c2c on
    z, bit for bit: the new state, the transformed lines and the
    divergence flag; fused kernels on power-of-two z, the two-kernel
    fallback otherwise."""
    import torch

    rng = np.random.default_rng(7 * kind + sum(shape))
    n0, n1, n2 = shape

    def cplx():
        return torch.from_numpy(rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).cuda()

    st = nat.stream_ptr()
    state, aux, aux2 = cplx(), cplx(), cplx()
    if kind == 2:
        state.view(-1)[len(state.view(-1)) // 2] = complex("nan")  # the flag must fire the same way
    kx, ky, kz = (torch.from_numpy(rng.standard_normal(m)).cuda() for m in shape)
    c = {0: (-0.3, 0.1, 0.0), 1: (0.1, 0.07, -2.0), 2: (1.0, 0.8, 0.1)}[kind]
    name = ("pfcs_hydro_psi_update_to", "pfcs_hydro_vel_update_to", "pfcs_ch_update_to")[kind]
    for a2 in ((aux2, None) if kind == 0 else (aux2,)):
        new_w = torch.empty_like(state)
        flag_w = torch.zeros(4096, dtype=torch.float64, device="cuda")
        ops = [nat.ptr(state), nat.ptr(new_w), nat.ptr(aux)] + ([] if kind == 1 else [nat.ptr(a2) if a2 is not None
                                                                                       else None])
        consts = c[:2] if kind == 0 else c
        nat.call(name, *ops, n0, n1, n2, nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), *consts, nat.ptr(flag_w), st)
        z_w = torch.empty_like(state)
        nat.call("pfcs_fft_axis_c2c", nat.ptr(new_w), nat.ptr(z_w), n0, n1, n2, 2, 0, st)
        new_g, z_g = torch.empty_like(state), torch.empty_like(state)
        flag_g = torch.zeros_like(flag_w)
        nat.call("pfcs_update_zinv", kind, nat.ptr(state), nat.ptr(aux), nat.ptr(a2) if a2 is not None else None,
                 nat.ptr(new_g), nat.ptr(z_g), n0, n1, n2, nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), *c,
                 nat.ptr(flag_g), st)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(new_g.cpu().numpy(), new_w.cpu().numpy())  # (NaN == NaN here)
        np.testing.assert_array_equal(z_g.cpu().numpy(), z_w.cpu().numpy())
        assert (flag_g.view(-1, 4)[:, 3].max() > 0) == (flag_w.view(-1, 4)[:, 3].max() > 0)


def test_update_zinv_argument_errors(nat):
    import torch

    x = torch.zeros((4, 4, 8), dtype=torch.complex128, device="cuda")
    k = torch.zeros(8, dtype=torch.float64, device="cuda")
    st = nat.stream_ptr()
    args = (nat.ptr(k), nat.ptr(k), nat.ptr(k), 1.0, 1.0, 1.0, None, st)
    with pytest.raises(Exception):  # unknown kind
        nat.call("pfcs_update_zinv", 3, nat.ptr(x), nat.ptr(x), None, nat.ptr(x), nat.ptr(x.clone()), 4, 4, 8, *args)
    with pytest.raises(Exception):  # zout aliasing the state
        nat.call("pfcs_update_zinv", 1, nat.ptr(x), nat.ptr(x.clone()), None, nat.ptr(x), nat.ptr(x), 4, 4, 8, *args)


@pytest.mark.parametrize("shape", [(9, 16, 512), (5, 12, 64), (6, 10, 9)])
@pytest.mark.parametrize("kind,flags", [(0, 1), (0, 2), (0, 3), (1, 1), (2, 3)])
def test_update_zzinv_bit_identical(nat, shape, kind, flags):
    """pfcs_update_zzinv (operands before their forward z pass, the z
    passes run inside the update) == the forward z passes, then
    pfcs_update_zinv — bit for bit; fused on power-of-two z, the in-place
    fallback otherwise."""
    import torch

    rng = np.random.default_rng(11 * kind + flags + sum(shape))
    n0, n1, n2 = shape

    def cplx():
        return torch.from_numpy(rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).cuda()

    st = nat.stream_ptr()
    state, aux, aux2 = cplx(), cplx(), cplx()
    kx, ky, kz = (torch.from_numpy(rng.standard_normal(m)).cuda() for m in shape)
    c = {0: (-0.3, 0.1, 0.0), 1: (0.1, 0.07, -2.0), 2: (1.0, 0.8, 0.1)}[kind]
    a_w, b_w = aux.clone(), aux2.clone()
    if flags & 1:
        nat.call("pfcs_fft_axis_c2c", nat.ptr(a_w), nat.ptr(a_w), n0, n1, n2, 2, 1, st)
    if flags & 2:
        nat.call("pfcs_fft_axis_c2c", nat.ptr(b_w), nat.ptr(b_w), n0, n1, n2, 2, 1, st)
    new_w, z_w = torch.empty_like(state), torch.empty_like(state)
    flag_w = torch.zeros(4096, dtype=torch.float64, device="cuda")
    nat.call("pfcs_update_zinv", kind, nat.ptr(state), nat.ptr(a_w), nat.ptr(b_w), nat.ptr(new_w), nat.ptr(z_w),
             n0, n1, n2, nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), *c, nat.ptr(flag_w), st)
    a_g, b_g = aux.clone(), aux2.clone()
    new_g, z_g = torch.empty_like(state), torch.empty_like(state)
    flag_g = torch.zeros_like(flag_w)
    nat.call("pfcs_update_zzinv", kind, nat.ptr(state), nat.ptr(a_g), nat.ptr(b_g), nat.ptr(new_g), nat.ptr(z_g),
             n0, n1, n2, nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), *c, flags, nat.ptr(flag_g), st)
    torch.cuda.synchronize()
    assert torch.equal(new_g, new_w)
    assert torch.equal(z_g, z_w)
