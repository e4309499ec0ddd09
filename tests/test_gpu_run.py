"""Run drivers on the GPU against the reference's own run outputs
(tests/golden/run_drivers.npz from oracle/gen_golden_run.py): diagnostics
rows, final fields and snapshot files of run_pfc (3D full volume and 2D
mid-plane slices) and run_hydro, plus decomposition invariance.

Tolerances: the north-star field bar (rel <= 1e-9) for fields after the
run; diagnostics rel <= 1e-9 (energies are sums over the grid); the mean
from the zero mode to 1e-12 absolute."""

import numpy as np
import pytest

from conftest import rel_inf

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_26818_b200 as p

    return p


def _diag(res, cols):
    return np.array([[row[c] for c in cols] for row in res.diagnostics], dtype=np.float64)


def _check_diag(got, want, tol=1e-9):
    assert got.shape == want.shape
    np.testing.assert_array_equal(got[:, 0], want[:, 0])  # step
    np.testing.assert_allclose(got[:, 1], want[:, 1], rtol=1e-14)  # time
    for c in range(2, got.shape[1]):
        scale = max(1.0, float(np.max(np.abs(want[:, c]))))
        assert float(np.max(np.abs(got[:, c] - want[:, c]))) <= tol * scale, (c, got[:, c], want[:, c])


@pytest.mark.parametrize("workers", [1, 2])
def test_run_pfc_3d_matches_reference(pkg, golden, tmp_path, workers):
    from paper_2603_26818_b200 import config, run, snapshot

    g = golden("run_drivers")
    cfg = config.load_config_dict({"grid": {"n": [32, 32, 32]}, "params": {"n_steps": 20}, "workers": workers,
                                   "io": {"out_dir": str(tmp_path), "diag_every": 5, "snap_every": 10,
                                          "full_volume": True}})
    res = run.run_pfc(cfg)
    _check_diag(_diag(res, run.PFC_COLUMNS[:-1]), g["pfc_diag"])
    assert len(res.realness) == 20
    assert rel_inf(res.final_psi, g["pfc_final"]) <= 1e-9
    hdr, snap10 = snapshot.read_snapshot(tmp_path / "psi_00000010_full.snap")
    assert hdr.step == 10 and abs(hdr.sim_time - 1.0) < 1e-12
    assert rel_inf(snap10, g["pfc_snap10"]) <= 1e-9
    meta = (tmp_path / "psi_00000010_full.snap.meta.txt").read_text()
    assert f"config_hash: {cfg.config_hash()}" in meta
    assert (tmp_path / "resolved_config.yaml").read_text() == cfg.resolved_yaml()
    lines = (tmp_path / "diagnostics.csv").read_text().splitlines()
    assert lines[0] == ",".join(run.PFC_COLUMNS) and len(lines) == 1 + len(res.diagnostics)
    names = sorted(p.name for p in tmp_path.glob("*.snap"))
    assert names == ["psi_00000000_full.snap", "psi_00000010_full.snap", "psi_00000020_full.snap"]


def test_run_pfc_decomposition_invariance(pkg, tmp_path):
    """Snapshots written by 1 and 3 ranks are byte-identical (the per-line
    arithmetic does not depend on the slab split)."""
    from paper_2603_26818_b200 import config, run

    outs = []
    for w in (1, 3):
        d = tmp_path / f"g{w}"
        cfg = config.load_config_dict({"grid": {"n": [24, 20, 18]}, "params": {"n_steps": 6}, "workers": w,
                                       "io": {"out_dir": str(d), "diag_every": 3, "snap_every": 6,
                                              "full_volume": True}})
        res = run.run_pfc(cfg)
        outs.append(((d / "psi_00000006_full.snap").read_bytes(), res.final_psi))
    assert outs[0][0] == outs[1][0]
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("workers", [1, 2])
def test_run_pfc_2d_slices_match_reference(pkg, golden, tmp_path, workers):
    from paper_2603_26818_b200 import config, run, snapshot

    g = golden("run_drivers")
    cfg = config.load_config_dict({"grid": {"n": [64, 48]}, "params": {"n_steps": 6}, "workers": workers,
                                   "init": {"kind": "single_mode_triangular_2d", "amplitude": 0.2},
                                   "io": {"out_dir": str(tmp_path), "diag_every": 3, "snap_every": 3,
                                          "full_volume": False}})
    res = run.run_pfc(cfg)
    _check_diag(_diag(res, run.PFC_COLUMNS[:-1]), g["pfc2_diag"])
    for name in ("slice_xy", "slice_xz", "slice_yz"):
        _, s = snapshot.read_snapshot(tmp_path / f"psi_00000006_{name}.snap")
        assert s.shape == g[f"pfc2_{name}"].shape
        assert rel_inf(s, g[f"pfc2_{name}"]) <= 1e-9, name


def test_run_hydro_serial_matches_reference(pkg, golden):
    from paper_2603_26818_b200 import config, run

    g = golden("run_drivers")
    cfg = config.load_config_dict({"model": "hydro", "grid": {"n": [16, 16, 16]},
                                   "params": {"n_steps": 4, "dt": 0.05},
                                   "init": {"seed": 4}, "io": {"diag_every": 1}})
    res = run.run_hydro(cfg)
    cols = [c for c in run.HYDRO_COLUMNS if c != "step_wall_seconds"]
    got = _diag(res, cols)
    want = g["hydro_diag"]
    _check_diag(got[:, :-1], want[:, :-1])
    np.testing.assert_allclose(got[:, -1], want[:, -1], atol=1e-13)  # mean drift ~ 1e-17
    assert rel_inf(res.final_psi, g["hydro_final_psi"]) <= 1e-9
    assert rel_inf(np.stack(res.final_v), g["hydro_final_v"]) <= 1e-9


def test_run_hydro_field_per_gpu_equals_serial(pkg):
    from paper_2603_26818_b200 import config, run

    base = {"model": "hydro", "grid": {"n": [16, 16, 16]}, "params": {"n_steps": 3, "dt": 0.05},
            "init": {"seed": 4}, "io": {"diag_every": 1}}
    r1 = run.run_hydro(config.load_config_dict(base))
    r4 = run.run_hydro(config.load_config_dict(dict(base, workers=4)))
    np.testing.assert_array_equal(r1.final_psi, r4.final_psi)
    for a, b in zip(r1.final_v, r4.final_v):
        np.testing.assert_array_equal(a, b)


def test_run_model_dispatch_and_divergence(pkg, tmp_path):
    from paper_2603_26818_b200 import config, pfc, run
    from paper_2603_26818_b200.transport import WorkerFailure

    res = run.run_model(config.load_config_dict({"grid": {"n": [16, 16, 16]}, "params": {"n_steps": 2}}))
    assert [r["step"] for r in res.diagnostics] == [0, 2]
    cfg = config.load_config_dict({"grid": {"n": [16, 16, 16]}, "params": {"n_steps": 30, "psi_bar": 1e110},
                                   "io": {"out_dir": str(tmp_path), "diag_every": 1}})
    with pytest.raises(WorkerFailure) as ei:  # as the reference: the worker's error, wrapped
        run.run_pfc(cfg)
    assert isinstance(ei.value.cause, pfc.DivergenceError) and ei.value.cause.step_index == 0
    rows = (tmp_path / "diagnostics.csv").read_text().splitlines()
    assert rows[0].startswith("step,time") and len(rows) >= 2  # partial series kept on disk
