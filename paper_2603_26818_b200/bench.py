"""PFC step-loop benchmark with per-worker field-memory accounting
(drop-in for the reference's ``pfcspectral.bench``, bench.py:1-160).

Same public surface and CSV schemas — ``FieldMemoryMeter``, ``BenchRow``,
``bench(config)``, ``write_bench_csv``, ``write_memory_csv`` — measured on
the device path:

* time: wall clock around ``n_steps`` fused steps per repetition, bracketed
  by a worker barrier and a device synchronisation on both sides (the
  device work is asynchronous, so the reference's bare ``perf_counter``
  would time only the enqueue);
* memory: ``baseline`` = the rank's spectral slab (``psi_hat``); each
  repetition samples the device buffers the step engine holds (receive /
  work slabs) plus the transients the distributed transforms sample
  (distfft.py exchange staging), so the peak is the per-rank device
  footprint of the step — what shrinks as 1/G.

This is the reference harness the acceptance suite drives
(test_acceptance.py:218-272); the repo's driver benchmark is the
top-level ``bench.py``.
"""

from __future__ import annotations

import csv
import statistics
import time
from dataclasses import dataclass
from pathlib import Path

import torch

from . import distfft, pfc
from .config import RunConfig
from .grid import make_symbols
from .transport import spawn_group

__all__ = ["FieldMemoryMeter", "BenchRow", "bench", "write_bench_csv", "write_memory_csv"]


class FieldMemoryMeter:
    """Peak of ``baseline + transient`` over all samples (never decreases)."""

    def __init__(self):
        self.baseline = 0
        self.peak = 0

    def sample(self, transient_bytes: int) -> None:
        self.peak = max(self.peak, self.baseline + int(transient_bytes))


@dataclass
class BenchRow:
    workers: int
    grid: str
    steps: int
    seconds_per_step_median: float
    seconds_per_step_min: float
    speedup_vs_g1: float
    peak_field_bytes_per_worker: int


def _engine_bytes(state: pfc.PfcState) -> int:
    """Distinct device buffers held by the rank's step engine."""
    eng = state._engine
    if eng is None:
        return 0
    seen, total = set(), 0
    for name in ("work", "send", "recv_z", "recv_x"):
        t = getattr(eng, name, None)
        if isinstance(t, torch.Tensor) and t.data_ptr() not in seen:
            seen.add(t.data_ptr())
            total += t.numel() * t.element_size()
    return total


def _run_once(config: RunConfig, workers: int, n_steps: int) -> tuple[float, int]:
    """One timed step loop on `workers` ranks: (seconds per step, peak bytes)."""
    grid, params, init = config.grid, config.pfc_params, config.init
    nx = grid.n[0]
    real = nx >= 4 and not (nx & (nx - 1))  # R2C path where the x kernels apply

    def body(worker):
        worker.meter = FieldMemoryMeter()
        lay = distfft._layout(grid, distfft.Layout.X_SLAB, worker.size, real)
        sym = make_symbols(grid, params.eps, layout=lay, rank=worker.rank)
        f0 = pfc.init_condition(init.kind, grid, worker, real=real, psi_bar=params.psi_bar, seed=init.seed,
                                noise_amplitude=init.noise_amplitude, amplitude=init.amplitude,
                                amplitude2=init.amplitude2, n_seeds=init.n_seeds,
                                seed_radius=init.seed_radius, on_incommensurate=init.on_incommensurate)
        state = pfc.PfcState(psi_hat=distfft.forward(f0, worker), grid=grid, symbols=sym, worker=worker)
        del f0
        psi = state.psi_hat.dev
        worker.meter.baseline = psi.numel() * psi.element_size()
        torch.cuda.synchronize(psi.device)
        worker.barrier()
        t0 = time.perf_counter()
        if n_steps > 0:
            pfc.pfc_run(state, params, n_steps)
        torch.cuda.synchronize(psi.device)
        worker.barrier()
        elapsed = time.perf_counter() - t0
        worker.meter.sample(_engine_bytes(state))
        return elapsed, worker.meter.peak

    res = spawn_group(workers, body)
    return max(r[0] for r in res) / max(n_steps, 1), max(r[1] for r in res)


def bench(config: RunConfig) -> list[BenchRow]:
    """Per worker count: warm-up run, then `repetitions` timed runs of
    `n_steps` steps (bench.py:95-123 semantics: median / min seconds per
    step, speedup vs the G = 1 median, per-worker peak field bytes)."""
    if config.bench.repetitions < 3:
        raise ValueError("bench needs repetitions >= 3")
    n_steps = config.pfc_params.n_steps
    label = "x".join(str(m) for m in config.grid.n)
    rows: list[BenchRow] = []
    g1 = None
    for workers in config.bench.workers_list:
        if config.bench.warmup_steps > 0:
            _run_once(config, workers, config.bench.warmup_steps)
        times, peak = [], 0
        for _ in range(config.bench.repetitions):
            t, p = _run_once(config, workers, n_steps)
            times.append(t)
            peak = max(peak, p)
        med = statistics.median(times)
        if g1 is None and workers == 1:
            g1 = med
        rows.append(BenchRow(workers=workers, grid=label, steps=n_steps, seconds_per_step_median=med,
                             seconds_per_step_min=min(times),
                             speedup_vs_g1=(g1 / med) if g1 else float("nan"),
                             peak_field_bytes_per_worker=peak))
    return rows


def write_bench_csv(rows: list[BenchRow], path: str | Path) -> Path:
    """G,grid,steps,seconds_per_step_median,seconds_per_step_min,speedup_vs_G1."""
    path = Path(path)
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["G", "grid", "steps", "seconds_per_step_median", "seconds_per_step_min", "speedup_vs_G1"])
        for r in rows:
            w.writerow([r.workers, r.grid, r.steps, repr(r.seconds_per_step_median),
                        repr(r.seconds_per_step_min), repr(r.speedup_vs_g1)])
    return path


def write_memory_csv(rows: list[BenchRow], path: str | Path) -> Path:
    """G,peak_field_bytes_per_worker,ratio_vs_G1."""
    path = Path(path)
    base = next((r.peak_field_bytes_per_worker for r in rows if r.workers == 1), None)
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["G", "peak_field_bytes_per_worker", "ratio_vs_G1"])
        for r in rows:
            w.writerow([r.workers, r.peak_field_bytes_per_worker,
                        repr(r.peak_field_bytes_per_worker / base if base else float("nan"))])
    return path
