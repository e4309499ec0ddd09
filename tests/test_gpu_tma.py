"""The TMA-staged passes (csrc/pfcs_tma.cu k_strided_tma; csrc/pfcs_x.cu
k_real_x with ST == 3) must be bit-identical to the register-pipelined kernels
they replace (PFCS_TMA=0): every tile width, ragged inner extents (OOB-filled
boxes), both directions, the real x transforms and the fused cube pass with
its diagnostics — including the line-synchronous cube pass k_cube_ls
(PFCS_CUBE_LS=0/1) at production tiles.

The switch is read once per process, so each configuration runs in a child
process that writes its outputs for comparison."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2603_26818_b200 import _native as nat
torch.cuda.set_device(0)
out = {{}}
for (outer, n, inner) in {cases!r}:
    rng = np.random.default_rng(n * 7 + inner)
    x = rng.standard_normal((outer, n, inner)) + 1j * rng.standard_normal((outer, n, inner))
    for fwd in (1, 0):
        a = torch.from_numpy(x).cuda()
        b = torch.empty_like(a)
        nat.call("pfcs_fft_axis_c2c", nat.ptr(a), nat.ptr(b), outer, n, inner, 1, fwd, nat.stream_ptr())
        ip = a.clone()
        nat.call("pfcs_fft_axis_c2c", nat.ptr(ip), nat.ptr(ip), outer, n, inner, 1, fwd, nat.stream_ptr())
        torch.cuda.synchronize()
        out[f"{{outer}}_{{n}}_{{inner}}_{{fwd}}"] = b.cpu().numpy()
        out[f"{{outer}}_{{n}}_{{inner}}_{{fwd}}_ip"] = ip.cpu().numpy()
for (n, inner) in {xcases!r}:
    rng = np.random.default_rng(n + inner)
    nh = n // 2 + 1
    r = torch.from_numpy(rng.standard_normal((n, inner))).cuda()
    h = torch.empty((nh, inner), dtype=torch.complex128, device="cuda")
    nat.call("pfcs_rfft_x", nat.ptr(r), nat.ptr(h), n, inner, nat.stream_ptr())
    r2 = torch.empty_like(r)
    nat.call("pfcs_irfft_x", nat.ptr(h), nat.ptr(r2), n, inner, nat.stream_ptr())
    c = h.clone()
    diag = torch.zeros(nat.DIAG_SLOTS * 4, dtype=torch.float64, device="cuda")
    nat.call("pfcs_pfc_cube_x", nat.ptr(c), n, inner, 1, nat.ptr(diag), nat.stream_ptr())
    torch.cuda.synchronize()
    out[f"x{{n}}_{{inner}}_r2c"] = h.cpu().numpy()
    out[f"x{{n}}_{{inner}}_c2r"] = r2.cpu().numpy()
    out[f"x{{n}}_{{inner}}_cube"] = c.cpu().numpy()
    out[f"x{{n}}_{{inner}}_diag"] = diag.cpu().numpy()
for (cx, ny, nz) in {zcases!r}:
    rng = np.random.default_rng(cx * ny + nz)
    shp = (cx, ny, nz)
    nl = torch.from_numpy(rng.standard_normal(shp) + 1j * rng.standard_normal(shp)).cuda()
    psi = torch.from_numpy(rng.standard_normal(shp) + 1j * rng.standard_normal(shp)).cuda()
    nxt = torch.empty_like(nl)
    kx = torch.linspace(0, 1, cx, dtype=torch.float64, device="cuda")
    ky = torch.linspace(0, 1, ny, dtype=torch.float64, device="cuda")
    kz = torch.linspace(0, 1, nz, dtype=torch.float64, device="cuda")
    diag = torch.zeros(nat.DIAG_SLOTS * 4, dtype=torch.float64, device="cuda")
    nat.call("pfcs_pfc_update_z", nat.ptr(nl), nat.ptr(psi), nat.ptr(nxt), cx, ny, nz, 1, 1,
             nat.ptr(kx), nat.ptr(ky), nat.ptr(kz), -0.3, 0.1, nat.ptr(diag), nat.stream_ptr())
    torch.cuda.synchronize()
    out[f"z{{cx}}_{{ny}}_{{nz}}_psi"] = psi.cpu().numpy()
    out[f"z{{cx}}_{{ny}}_{{nz}}_next"] = nxt.cpu().numpy()
    out[f"z{{cx}}_{{ny}}_{{nz}}_diag"] = diag.cpu().numpy()
np.savez({path!r}, **out)
"""

ZCASES = [(3, 5, 256), (2, 7, 1024), (5, 3, 64), (4, 4, 512)]
# (1024, 3000) and (2048, 1000): production tiles of the line-synchronous cube
# pass k_cube_ls (PFCS_TMA=1) against the register-pipelined k_real_x
XCASES = [(128, 96), (256, 1000), (512, 1030), (1024, 520), (1024, 64), (1024, 3000), (2048, 1000)]
CASES = [(3, 64, 40), (2, 128, 33), (2, 256, 16), (2, 512, 9), (3, 1024, 12), (1, 2048, 5), (2, 1024, 1000)]


def _run(tmp_path, name, env):
    path = str(tmp_path / f"{name}.npz")
    code = CHILD.format(root=str(ROOT), cases=CASES, xcases=XCASES, zcases=ZCASES, path=path)
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, "-c", code], check=True, env=e, timeout=300)
    return np.load(path)


@pytest.mark.parametrize("t", [1, 2, 4, 8])
def test_tma_strided_bit_identical(tmp_path, t):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    base = _run(tmp_path, "base", {"PFCS_TMA": "0"})
    tma = _run(tmp_path, f"tma{t}", {"PFCS_TMA": "1", "PFCS_TMA_T": str(t)})
    for k in base.files:
        assert np.array_equal(base[k], tma[k]), k


def test_cube_ls_bit_identical(tmp_path):
    """k_cube_ls (line-synchronous, TMA load + store) reproduces the
    interleaved-tile TMA cube pass k_real_x<M, T, 3, MODE_CUBE> bit for bit,
    incl. ragged last tiles and the max|psi| diagnostic."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a = _run(tmp_path, "ls1", {"PFCS_CUBE_LS": "1"})
    b = _run(tmp_path, "ls0", {"PFCS_CUBE_LS": "0"})
    keys = [k for k in a.files if k.startswith("x")]
    assert any(k.startswith("x1024_3000") for k in keys)
    for k in keys:
        assert np.array_equal(a[k], b[k]), k
