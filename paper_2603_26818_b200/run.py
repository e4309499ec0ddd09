"""Run drivers: PFC and hydro time loops with diagnostics and snapshots
(reference /root/reference/pkg/src/pfcspectral/run.py).

Same entry points and outputs as the reference: ``run_pfc(config)``,
``run_hydro(config)``, ``run_model(config)`` return a ``RunResult`` with the
rank-0 diagnostics rows; with ``io.out_dir`` set they write
``resolved_config.yaml``, ``diagnostics.csv`` (columns ``PFC_COLUMNS`` /
``HYDRO_COLUMNS``, flushed row by row so a divergence leaves the partial
series) and PFCSNAP1 snapshots ``psi_<step:08d>_<full|slice_xy|slice_xz|slice_yz>.snap``.

B200-native differences (same numbers, different plumbing):

* the PFC loop runs ``pfc.pfc_run`` between diagnostic/snapshot events (steps
  enqueued back to back, one device->host read per chunk) instead of one
  host round trip per step; ``step_wall_seconds`` is the chunk's wall time
  per step and ``RunResult.realness`` still has one entry per step;
* the PFC state is the R2C half spectrum of a real field (``real=True``, the
  default, for power-of-two nx; otherwise, or with ``real=False``, the
  reference's complex128 path on the C2C kernels);
* initial conditions are built slab by slab on each rank
  (``pfc.initial_field_slab``), and full-volume snapshots are written by all
  ranks in parallel from their device slabs (``snapshot.write_snapshot_slabs``)
  — neither ever materialises the full field on one rank; mid-plane slices
  are assembled on rank 0 from the ranks' pieces;
* ``final_psi`` (the gathered field the reference returns) is only
  assembled up to ``FINAL_GATHER_MAX_POINTS``.
"""

from __future__ import annotations

import csv
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import distfft, hydro, pfc
from .config import RunConfig
from .distfft import Space
from .grid import make_symbols
from .snapshot import write_snapshot, write_snapshot_slabs
from .transport import spawn_group

__all__ = ["RunResult", "run_pfc", "run_hydro", "run_model", "PFC_COLUMNS", "HYDRO_COLUMNS"]

PFC_COLUMNS = ["step", "time", "free_energy", "mean_psi", "max_abs_psi", "step_wall_seconds"]
HYDRO_COLUMNS = PFC_COLUMNS + ["max_abs_v1", "max_abs_v2", "max_abs_v3", "mean_psi_drift"]

FULL_SNAPSHOT_MAX_POINTS = 128 ** 3  # auto full-volume snapshots up to this size (run.py:37)
FINAL_GATHER_MAX_POINTS = 1 << 27  # 1 GiB of float64


@dataclass
class RunResult:
    diagnostics: list = field(default_factory=list)
    snapshot_paths: list = field(default_factory=list)
    final_psi: np.ndarray | None = None
    final_v: list | None = None
    realness: list = field(default_factory=list)  # per step max|Im psi| / max|Re psi|
    diverged: bool = False


class _Diagnostics:
    """Rows kept in memory and appended to a CSV as they arrive."""

    def __init__(self, path: Path | None, columns: list):
        self.rows: list = []
        self._fh = open(path, "w", newline="") if path else None
        self._w = None
        if self._fh:
            self._w = csv.DictWriter(self._fh, fieldnames=columns)
            self._w.writeheader()
            self._fh.flush()

    def add(self, row: dict) -> None:
        self.rows.append(row)
        if self._w:
            self._w.writerow(row)
            self._fh.flush()

    def close(self) -> None:
        if self._fh:
            self._fh.close()
            self._fh = None


def _out_dir(config: RunConfig) -> Path | None:
    if config.io.out_dir is None:
        return None
    out = Path(config.io.out_dir)
    out.mkdir(parents=True, exist_ok=True)
    (out / "resolved_config.yaml").write_text(config.resolved_yaml())
    return out


def _full_volume(config: RunConfig) -> bool:
    if config.io.full_volume is not None:
        return bool(config.io.full_volume)
    return config.grid.num_points <= FULL_SNAPSHOT_MAX_POINTS


def _slice_piece(local: torch.Tensor, lay, rank: int, fixed_axis: int, index: int):
    """This rank's part of the global mid-plane slice {fixed_axis = index}
    (None when the slab does not intersect it); 3D with a unit fixed axis."""
    if fixed_axis == lay.axis:
        lo = lay.offsets[rank]
        if not (lo <= index < lo + lay.counts[rank]):
            return None
        index -= lo
    sl = [slice(None)] * 3
    sl[fixed_axis] = slice(index, index + 1)
    return local[tuple(sl)].double().cpu().numpy()


def _gather_slices(phys, worker) -> dict | None:
    """Mid-plane slices of a physical slab field, assembled on rank 0 as the
    reference's ``_snapshot_fields`` returns them (run.py:80-89)."""
    grid = phys.grid
    nx, ny, nz = grid.shape
    lay = distfft.layout_for(grid, phys.layout, worker.size)
    local = phys.dev.real if phys.dev.is_complex() else phys.dev
    specs = [("slice_xy", 2, nz // 2), ("slice_xz", 1, ny // 2), ("slice_yz", 0, nx // 2)]
    mine = [_slice_piece(local, lay, worker.rank, ax, idx) for _, ax, idx in specs]
    everyone = worker.all_to_all([mine] * worker.size)  # rank r receives every rank's pieces
    if worker.rank != 0:
        return None
    out = {}
    for k, (name, ax, _) in enumerate(specs):
        parts = [everyone[r][k] for r in range(worker.size) if everyone[r][k] is not None]
        out[name] = parts[0] if ax == lay.axis else np.concatenate(parts, axis=lay.axis)
    return out


def _snapshot(out: Path, prefix: str, psi_hat, worker, step: int, sim_time: float, config: RunConfig,
              paths: list) -> None:
    """Collective: inverse transform + full-volume (parallel) or slices (rank 0)."""
    meta = {"config_hash": config.config_hash()}
    phys = distfft.inverse(psi_hat, worker)
    if _full_volume(config):
        path = out / f"{prefix}_{step:08d}_full.snap"
        write_snapshot_slabs(path, phys, worker, step, sim_time, meta=meta)
        if worker.rank == 0:
            paths.append(path)
        return
    slices = _gather_slices(phys, worker)
    if worker.rank == 0:
        for name, data in slices.items():
            path = out / f"{prefix}_{step:08d}_{name}.snap"
            write_snapshot(path, data, step, sim_time, meta=meta)
            paths.append(path)


def _final_field(psi_hat, worker, grid):
    if grid.num_points > FINAL_GATHER_MAX_POINTS:
        return None
    return np.asarray(distfft.gather(distfft.inverse(psi_hat, worker), worker).real)


def _events(n_steps: int, diag_every: int, snap_every: int | None) -> list:
    """Steps after which the loop stops for diagnostics/snapshots."""
    ev = {n_steps}
    ev.update(range(diag_every, n_steps + 1, diag_every))
    if snap_every:
        ev.update(range(snap_every, n_steps + 1, snap_every))
    return sorted(e for e in ev if e >= 1)


def run_pfc(config: RunConfig, *, real: bool = True) -> RunResult:
    """Slab-decomposed PFC run per the config (run.py:113-184); returns the
    rank-0 result."""
    grid = config.grid
    params = config.pfc_params
    init = config.init
    out = _out_dir(config)

    nx = grid.n[0]
    use_real = real and nx >= 4 and not (nx & (nx - 1))  # R2C kernels need a power-of-two nx

    def body(worker) -> RunResult | None:
        half = use_real
        xlay = distfft._layout(grid, distfft.Layout.X_SLAB, worker.size, half)
        sym = make_symbols(grid, params.eps, layout=xlay, rank=worker.rank)
        f0 = pfc.init_condition(init.kind, grid, worker, real=use_real, psi_bar=params.psi_bar, seed=init.seed,
                                noise_amplitude=init.noise_amplitude, amplitude=init.amplitude,
                                amplitude2=init.amplitude2, n_seeds=init.n_seeds,
                                seed_radius=init.seed_radius, on_incommensurate=init.on_incommensurate)
        state = pfc.PfcState(psi_hat=distfft.forward(f0, worker), grid=grid, symbols=sym, worker=worker)
        del f0
        root = worker.rank == 0
        diag = _Diagnostics(out / "diagnostics.csv" if (out and root) else None, PFC_COLUMNS)
        result = RunResult(diagnostics=diag.rows)

        def record(wall: float) -> None:
            energy = pfc.free_energy(state, params)
            mean_psi, max_abs = pfc.mean_and_max(state)
            diag.add({"step": state.step_index, "time": state.sim_time, "free_energy": energy,
                      "mean_psi": mean_psi, "max_abs_psi": max_abs, "step_wall_seconds": wall})

        try:
            record(0.0)
            if out is not None:
                _snapshot(out, "psi", state.psi_hat, worker, state.step_index, state.sim_time, config,
                          result.snapshot_paths)
            done = 0
            for ev in _events(params.n_steps, config.io.diag_every,
                              config.io.snap_every if out is not None else None):
                # steps before the last one of the block run back to back;
                # step_wall_seconds is the wall time of the single step just
                # before the diagnostic row, as in the reference (run.py:166-169)
                if ev - done > 1:
                    pfc.pfc_run(state, params, ev - done - 1, realness=result.realness)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                pfc.pfc_run(state, params, 1, realness=result.realness)
                wall = time.perf_counter() - t0
                done = ev
                if ev % config.io.diag_every == 0 or ev == params.n_steps:
                    record(wall)
                if out is not None and ev % config.io.snap_every == 0:
                    _snapshot(out, "psi", state.psi_hat, worker, state.step_index, state.sim_time, config,
                              result.snapshot_paths)
        except pfc.DivergenceError:
            result.diverged = True
            diag.close()
            raise
        result.final_psi = _final_field(state.psi_hat, worker, grid)
        diag.close()
        return result if root else None

    return spawn_group(config.workers, body)[0]


def _hydro_record(diag, result, step, sim_time, psi, v, sym, grid, wall, mean0, every, n_steps):
    """One hydro diagnostics row (run.py:210-229) from device fields."""
    pr = psi.real
    max_abs = float(pr.abs().max())
    max_imag = float(psi.imag.abs().max())
    result.realness.append(max_imag / max_abs if max_abs else 0.0)
    if step % every == 0 or step in (0, n_steps):
        mean = float(pr.mean())
        diag.add({"step": step, "time": sim_time, "free_energy": hydro.free_energy_full(psi, sym, grid),
                  "mean_psi": mean, "max_abs_psi": max_abs, "step_wall_seconds": wall,
                  "max_abs_v1": float(v[0].real.abs().max()), "max_abs_v2": float(v[1].real.abs().max()),
                  "max_abs_v3": float(v[2].real.abs().max()), "mean_psi_drift": mean - mean0})


def run_hydro(config: RunConfig) -> RunResult:
    """Hydrodynamic PFC run: serial dataflow on one GPU (workers = 1) or the
    field-per-GPU split (workers = 4: density on rank 0, v_i on rank i)
    (run.py:187-304).  Fields are device-resident full grids."""
    grid = config.grid
    hparams = config.hydro_params
    if hparams is None:
        raise ValueError("run_hydro needs hydro params (model: hydro)")
    params = hparams.pfc
    init = config.init
    out = _out_dir(config)
    psi0 = pfc.initial_field(init.kind, grid, psi_bar=params.psi_bar, seed=init.seed,
                             noise_amplitude=init.noise_amplitude, amplitude=init.amplitude,
                             amplitude2=init.amplitude2, n_seeds=init.n_seeds, seed_radius=init.seed_radius,
                             on_incommensurate=init.on_incommensurate)
    mean0 = float(psi0.mean())
    every = config.io.diag_every

    def snap(result, step, sim_time, psi):
        if out is None:
            return
        data = psi.real.cpu().numpy()
        meta = {"config_hash": config.config_hash()}
        if _full_volume(config):
            items = [("full", data)]
        else:
            nx, ny, nz = data.shape
            items = [("slice_xy", data[:, :, nz // 2][:, :, None]), ("slice_xz", data[:, ny // 2, :][:, None, :]),
                     ("slice_yz", data[nx // 2, :, :][None, :, :])]
        for name, block in items:
            path = out / f"psi_{step:08d}_{name}.snap"
            write_snapshot(path, block, step, sim_time, meta=meta)
            result.snapshot_paths.append(path)

    def initial(dev):
        sym = make_symbols(grid, params.eps, a0=hparams.a0)
        p = torch.as_tensor(psi0, dtype=torch.complex128, device=dev)
        psi_hat = hydro._fft(p, True)
        return sym, psi_hat, hydro._fft(psi_hat, False)

    if config.workers == 1:
        dev = torch.device("cuda", torch.cuda.current_device())
        sym, psi_hat, psi = initial(dev)
        zeros = lambda: torch.zeros(grid.shape, dtype=torch.complex128, device=dev)  # noqa: E731
        fields = hydro.HydroFields(psi_hat=psi_hat, psi=psi, v_hat=[zeros() for _ in range(3)],
                                   v=[zeros() for _ in range(3)])
        diag = _Diagnostics(out / "diagnostics.csv" if out else None, HYDRO_COLUMNS)
        result = RunResult(diagnostics=diag.rows)
        try:
            _hydro_record(diag, result, 0, 0.0, fields.psi, fields.v, sym, grid, 0.0, mean0, every, params.n_steps)
            snap(result, 0, 0.0, fields.psi)
            for step in range(1, params.n_steps + 1):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                hydro.serial_hydro_step(fields, sym, hparams)
                torch.cuda.synchronize()
                wall = time.perf_counter() - t0
                _hydro_record(diag, result, step, fields.sim_time, fields.psi, fields.v, sym, grid, wall, mean0,
                              every, params.n_steps)
                if out is not None and step % config.io.snap_every == 0:
                    snap(result, step, fields.sim_time, fields.psi)
        except pfc.DivergenceError:
            result.diverged = True
            diag.close()
            raise
        result.final_psi = fields.psi.real.cpu().numpy()
        result.final_v = [v.real.cpu().numpy() for v in fields.v]
        diag.close()
        return result

    if config.workers != 4:
        raise ValueError("hydro runs need exactly 1 or 4 workers")

    def body(worker) -> RunResult | None:
        dev = worker.device if getattr(worker, "device", None) is not None else torch.device("cuda")
        sym, psi_hat, psi = initial(dev)
        zeros = lambda: torch.zeros(grid.shape, dtype=torch.complex128, device=dev)  # noqa: E731
        if worker.rank == 0:
            role = {"psi_hat": psi_hat, "psi": psi, "v": [zeros() for _ in range(3)], "step_index": 0}
        else:
            role = {"v_hat": zeros(), "v_own": zeros(), "psi": psi, "step_index": 0}
        root = worker.rank == 0
        diag = _Diagnostics(out / "diagnostics.csv" if (out and root) else None, HYDRO_COLUMNS)
        result = RunResult(diagnostics=diag.rows)
        try:
            if root:
                _hydro_record(diag, result, 0, 0.0, role["psi"], role["v"], sym, grid, 0.0, mean0, every,
                              params.n_steps)
                snap(result, 0, 0.0, role["psi"])
            for step in range(1, params.n_steps + 1):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                hydro.parallel_hydro_step(worker, role, sym, hparams)
                torch.cuda.synchronize()
                wall = time.perf_counter() - t0
                if root:
                    _hydro_record(diag, result, step, step * params.dt, role["psi"], role["v"], sym, grid, wall,
                                  mean0, every, params.n_steps)
                    if out is not None and step % config.io.snap_every == 0:
                        snap(result, step, step * params.dt, role["psi"])
        except pfc.DivergenceError:
            result.diverged = True
            diag.close()
            raise
        diag.close()
        if root:
            result.final_psi = role["psi"].real.cpu().numpy()
            result.final_v = [v.real.cpu().numpy() for v in role["v"]]
            return result
        return None

    return spawn_group(4, body)[0]


def run_model(config: RunConfig) -> RunResult:
    """Dispatch on ``config.model`` (run.py:307-310)."""
    if config.model == "hydro":
        return run_hydro(config)
    return run_pfc(config)
