"""Host-side logic on CPU: the C ABI library, grid/symbol bookkeeping,
initial conditions, the in-process transport (reference test_transport.py
semantics) and the no-fallback rule."""

import math
import re
import time
from pathlib import Path

import numpy as np
import pytest

import ref_numpy as ora

ROOT = Path(__file__).resolve().parent.parent


# ------------------------------------------------------------------ C ABI ----

def test_library_exports_every_header_symbol():
    import ctypes

    from paper_2603_26818_b200 import _native

    lib = _native.load(require_cuda=False)
    header = (ROOT / "include" / "pfcs.h").read_text()
    declared = set(re.findall(r"^(?:int|int64_t|const char\*)\s+(pfcs_\w+)\(", header, re.M))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_native.exported_symbols())
    assert lib.pfcs_version() == 100
    so = ctypes.CDLL(str(_native.LIB_PATH))
    assert so.pfcs_last_error is not None


def test_no_cpu_fallback():
    import torch

    import paper_2603_26818_b200 as p

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        p.fft_nd(np.zeros((2, 2, 2)))


def test_kernel_sources_target_sm100a():
    from paper_2603_26818_b200 import _build

    assert "arch=compute_100a,code=sm_100a" in " ".join(_build.ARCH)
    assert _build.LIB.exists()


# ------------------------------------------------------------------- grid ----

def test_wavenumbers_and_layouts():
    from paper_2603_26818_b200.grid import GridSpec, slab_layout, wavenumbers

    for n in range(1, 17):
        g = GridSpec((n, 1, 1), (3.7, 1.0, 1.0))
        np.testing.assert_array_equal(wavenumbers(g, 0), ora.wavenumbers(n, 3.7))
    assert slab_layout(7, 4).counts == (2, 2, 2, 1)
    assert slab_layout(7, 4).offsets == (0, 2, 4, 6)
    assert slab_layout(2, 4).counts == (1, 1, 0, 0)
    for n, g in [(1, 1), (5, 2), (16, 3), (3, 7), (12, 4), (513, 8)]:
        lay = slab_layout(n, g)
        assert list(lay.counts) == ora.slab_counts(n, g)
    with pytest.raises(ValueError):
        slab_layout(4, 0)
    with pytest.raises(ValueError):
        GridSpec((0, 4, 4), (1.0, 1.0, 1.0))


def test_symbols_bit_identical_to_reference_formulas():
    from paper_2603_26818_b200.grid import GridSpec, make_symbols, slab_layout

    n = (12, 10, 8)
    L = (2 * math.pi * math.sqrt(3), 5.0, 7.5)
    grid = GridSpec(n, L)
    sym = make_symbols(grid, -0.3, a0=2.0)
    want = ora.symbols(n, L, -0.3, a0=2.0)
    for k in ("lap", "two_ring", "op", "linear", "cg", "d1", "d2", "d3"):
        np.testing.assert_array_equal(getattr(sym, k), want[k])
    lay = slab_layout(12, 3, axis=0)
    parts = [make_symbols(grid, -0.3, layout=lay, rank=r).lap for r in range(3)]
    np.testing.assert_array_equal(np.concatenate(parts, axis=0), want["lap"])
    assert np.all(sym.d1.real == 0.0)
    with pytest.raises(ValueError):
        make_symbols(grid, eps=math.nan)


def test_initial_fields_bit_identical_to_reference(golden):
    from paper_2603_26818_b200.grid import GridSpec
    from paper_2603_26818_b200.pfc import default_domain_length, initial_field

    g = golden("init")
    g3 = GridSpec((8, 8, 8), (2 * math.pi * math.sqrt(3),) * 3)
    g2 = GridSpec((32, 32, 1), default_domain_length((32, 32, 1)))
    np.testing.assert_array_equal(initial_field("constant_plus_noise", g3, seed=42), g["noise"])
    np.testing.assert_array_equal(initial_field("seeded_crystallites", g3, seed=42, n_seeds=3),
                                  g["crystallites"])
    np.testing.assert_array_equal(initial_field("two_mode_fcc_3d", g3, amplitude=0.07), g["fcc"])
    np.testing.assert_array_equal(
        initial_field("single_mode_triangular_2d", g2, amplitude=0.3, psi_bar=-0.2), g["tri"])
    np.testing.assert_array_equal(initial_field("seeded_crystallites", g2, seed=7, n_seeds=2),
                                  g["tri_seeds"])
    for name in ("pfc2d_256", "pfc3d_32"):
        run = golden(name)
        n = run["init"].shape
        grid = GridSpec(n, tuple(run["length"]))
        np.testing.assert_array_equal(
            initial_field("constant_plus_noise", grid, psi_bar=-0.3, seed=0, noise_amplitude=0.01),
            run["init"])
    with pytest.raises(ValueError, match="unknown init kind"):
        initial_field("bogus", g3)


# -------------------------------------------------------------- transport ----

def test_spawn_group_and_messaging():
    from paper_2603_26818_b200.transport import spawn_group

    assert spawn_group(4, lambda w: w.rank**2) == [0, 1, 4, 9]

    def body(w):
        if w.rank == 0:
            w.send(1, 9, "a")
            w.send(1, 9, "b")
            w.send(1, 4, np.array([1.0, 2.0]))
            return None
        return [w.receive(0, 9), w.receive(0, 9), w.receive(0, 4)]

    out = spawn_group(2, body)[1]
    assert out[:2] == ["a", "b"]
    np.testing.assert_array_equal(out[2], [1.0, 2.0])


def test_failure_attribution_and_timeouts():
    from paper_2603_26818_b200.transport import (DeadlockError, TransportError, WorkerFailure,
                                                 spawn_group)

    def body(w):
        if w.rank == 2:
            raise RuntimeError("boom")
        w.barrier()

    with pytest.raises(WorkerFailure) as info:
        spawn_group(3, body, timeout=5.0)
    assert info.value.rank == 2 and "boom" in str(info.value)

    def lonely(w):
        w.receive(1, 3)

    t0 = time.time()
    with pytest.raises(WorkerFailure) as info:
        spawn_group(2, lonely, timeout=0.3)
    assert isinstance(info.value.cause, (DeadlockError, TransportError))
    assert time.time() - t0 < 10
    with pytest.raises(ValueError):
        spawn_group(0, lambda w: None)


def test_all_to_all_and_barrier_generations():
    from paper_2603_26818_b200.transport import spawn_group

    def body(w):
        out = w.all_to_all([(w.rank, h) for h in range(w.size)])
        for _ in range(200):
            w.barrier()
        return out

    res = spawn_group(3, body)
    for r, got in enumerate(res):
        assert got == [(g, r) for g in range(3)]


def test_rank_ordered_reduction_identical_on_all_ranks():
    from paper_2603_26818_b200.pfc import _reduce_max, _reduce_sum
    from paper_2603_26818_b200.transport import spawn_group

    vals = [0.1, 1e16, -1e16, 0.3]

    def body(w):
        return _reduce_sum(w, vals[w.rank]), _reduce_max(w, vals[w.rank])

    res = spawn_group(4, body)
    assert len(set(res)) == 1
    total = 0.0
    for v in vals:
        total += v
    assert res[0][0] == total
