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
