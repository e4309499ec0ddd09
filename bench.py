#!/usr/bin/env python
"""Benchmark of the B200 pseudo-spectral hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 runs in-process; N > 1 is launched by torchrun (one process per GPU,
NCCL all-to-all over NVLink).  Headline (BASELINE.json configs[1]):

  metric  "distributed 3D FFT GB/s (fp64)"
  step    one forward + inverse distributed transform of a real 512^3 fp64
          field (R2C/C2R, slab decomposition), input resident in HBM
  value   algorithmic HBM bytes of the round trip / device time, whole job
          (2 x (R + 5S), R = 8 N^3, S = 16 N^2 (N/2+1))
  e2e     the same step through the public API (distfft.forward/inverse)
          with the field copied host->device before and device->host after,
          inside the timed region
  pfc     the other half of the metric: PFC time-steps/s on 1024^3 (R2C,
          fused passes), same timing rules, roofline 10 S per step

`--impl reference` times the reference algorithm on the host cores instead
(the oracle's restatement of distfft.py over a thread worker group — the
reference is a pure-Python package and does not travel to the GPU box).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FFT_N = 512
PFC_N = 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--fft-n", type=int, default=FFT_N)
    ap.add_argument("--pfc-n", type=int, default=PFC_N)
    ap.add_argument("--no-pfc", action="store_true")
    ap.add_argument("--pfc-big", action="store_true", help="also run the 2048^3 PFC step on one GPU")
    ap.add_argument("--pfc-big-n", type=int, default=2048)
    ap.add_argument("--multi-n", type=int, default=512)
    ap.add_argument("--no-multi", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    return ap.parse_args()


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fft_bytes(n: int) -> float:
    R = 8.0 * n**3
    S = 16.0 * n * n * (n // 2 + 1)
    return 2.0 * (R + 5.0 * S)


def pfc_bytes(n: int) -> float:
    return 10.0 * 16.0 * n * n * (n // 2 + 1)


def kernel_bytes(name: str, args) -> float:
    """Algorithmic HBM bytes of one libpfcs launch (read + write once)."""
    if name in ("pfcs_rfft_x", "pfcs_irfft_x"):
        nx, inner = args[2], args[3]
        return nx * inner * 8.0 + (nx // 2 + 1) * inner * 16.0
    if name == "pfcs_fft_axis_c2c":
        return 2.0 * 16.0 * args[2] * args[3] * args[4]
    if name == "pfcs_fft_zlines":
        return 2.0 * 16.0 * args[2] * args[3]
    if name == "pfcs_pfc_cube_x":
        nx, inner, real = args[1], args[2], args[3]
        return 2.0 * 16.0 * (nx // 2 + 1 if real else nx) * inner
    if name in ("pfcs_pfc_update_z", "pfcs_pfc_update_z_to"):
        return 4.0 * 16.0 * args[3] * args[4] * args[5]
    if name == "pfcs_fft_zlines_to":  # fused-exchange forms: same HBM bytes, stores go to peers
        return 2.0 * 16.0 * args[2] * args[3]
    if name == "pfcs_fft_lines_scatter":
        return 2.0 * 16.0 * args[2] * args[3] * args[4]
    return 0.0


def kernel_label(name: str, args) -> str:
    if name == "pfcs_fft_axis_c2c":
        return f"fft_axis{args[5]}_{'fwd' if args[6] else 'inv'}"
    if name == "pfcs_fft_zlines":
        return f"fft_z_{'fwd' if args[6] else 'inv'}"
    return name.replace("pfcs_", "")


class ClockSampler:
    """nvidia-smi sampling of SM clocks / throttle reasons during a region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------- helpers --

class Ctx:
    def __init__(self, n_gpus: int):
        import torch

        self.torch = torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != n_gpus and not (self.world == 1 and n_gpus == 1):
            if self.world == 1 and n_gpus > 1:
                raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist

            # PFCS_BENCH_BACKEND=gloo (test only): host-staged exchanges, ranks may
            # share a GPU — used to exercise the multi-rank path on a 1-GPU box
            backend = os.environ.get("PFCS_BENCH_BACKEND", "nccl")
            dev = self.local % torch.cuda.device_count()
            torch.cuda.set_device(dev)
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
            else:
                dist.init_process_group(backend)
            self.dist = dist
        else:
            torch.cuda.set_device(0)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.coll_device = self.device if (self.dist is None or self.dist.get_backend() == "nccl") else "cpu"

    def worker(self):
        from paper_2603_26818_b200.transport import ProcessWorker, Worker, WorkerGroup

        if self.world > 1:
            return ProcessWorker(device=self.device)
        return Worker(WorkerGroup(1), 0, self.device)

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max_over_ranks(self, v: float) -> float:
        if self.dist is None:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.coll_device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, v: float) -> float:
        if self.dist is None:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.coll_device)
        self.dist.all_reduce(t)
        return float(t.item())


def timed(ctx, fn, steps: int, warmup: int, drain=None):
    """W untimed steps, then K steps bracketed by barrier + synchronize on
    both sides, device time from CUDA events, max over ranks (ms/step).
    `drain()` (if given) makes the current stream wait for any side streams
    the steps used, so the end event covers their work too."""
    torch = ctx.torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ctx.barrier()
    torch.cuda.synchronize()
    from paper_2603_26818_b200 import _native as nat

    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    n0 = nat.launches
    a.record()
    for _ in range(steps):
        fn()
    if drain is not None:
        drain()
    b.record()
    torch.cuda.synchronize()
    ctx.timed_launches = nat.launches - n0  # libpfcs launches inside the timed region
    ctx.barrier()
    torch.cuda.synchronize()
    return ctx.max_over_ranks(a.elapsed_time(b) / steps)


def kernel_table(trace, steps):
    agg = {}
    for name, args, a, b in trace:
        lab = kernel_label(name, args)
        ms = a.elapsed_time(b)
        d = agg.setdefault(lab, {"launches": 0, "ms": 0.0, "bytes": 0.0})
        d["launches"] += 1
        d["ms"] += ms
        d["bytes"] += kernel_bytes(name, args)
    out = {}
    for lab, d in agg.items():
        avg = d["ms"] / d["launches"]
        out[lab] = {"launches_per_step": d["launches"] / steps, "avg_ms": round(avg, 4),
                    "alg_gb_per_launch": round(d["bytes"] / d["launches"] / 1e9, 4),
                    "gbs": round(d["bytes"] / d["launches"] / (avg * 1e-3) / 1e9, 1) if avg > 0 else None}
    return out


def measured_traffic(workload: str) -> dict:
    """DRAM read+write bytes per launch from the committed ncu --set full
    capture of the same workload (profiles/*_traffic.json), if any."""
    best = {}
    for p in sorted((ROOT / "profiles").glob("*_traffic.json")):
        try:
            d = json.loads(p.read_text())
        except Exception:
            continue
        if d.get("workload") == workload:
            best = d.get("traffic_bytes_per_launch", {})
    return best


def roofline_of(table, peak, peak_kind, traffic_map=None):
    top = max(table.items(), key=lambda kv: kv[1]["avg_ms"] * kv[1]["launches_per_step"])
    lab, d = top
    traffic = (traffic_map or {}).get(lab)
    return {"kernel": lab, "bound": "hbm", "achieved": d["gbs"], "peak": peak, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": round(d["gbs"] / peak, 4) if d["gbs"] else None,
            "traffic": traffic, "alg_bytes_per_launch": d["alg_gb_per_launch"] * 1e9}


# ------------------------------------------------------------ our workloads --

def run_fft(ctx, args, out):
    import torch

    from paper_2603_26818_b200 import _native as nat
    from paper_2603_26818_b200 import distfft
    from paper_2603_26818_b200.grid import GridSpec, slab_layout

    n = args.fft_n
    w = ctx.worker()
    grid = GridSpec((n, n, n), (1.0, 1.0, 1.0))
    cz = slab_layout(n, ctx.world).counts[ctx.rank]
    gen = torch.Generator(device=ctx.device).manual_seed(1234 + ctx.rank)
    x = torch.randn((n, n, cz), dtype=torch.float64, device=ctx.device, generator=gen)
    field = distfft.DistField(grid, distfft.Layout.Z_SLAB, distfft.Space.PHYSICAL, x)
    holder = {}

    def step():
        spec = distfft.forward(field, w)
        holder["back"] = distfft.inverse(spec, w)

    ms = timed(ctx, step, args.steps, args.warmup)
    launches = ctx.timed_launches
    # per-kernel device times over a traced pass of the same K steps
    nat.trace = []
    timed(ctx, step, args.steps, 0)
    table = kernel_table(nat.trace, args.steps)
    nat.trace = None
    # parity of the last round trip (size-independent property)
    err = float(torch.linalg.vector_norm(holder["back"].dev - x) / torch.linalg.vector_norm(x))
    err = ctx.max_over_ranks(err)

    # e2e through the public API with host buffers: every step copies its
    # input field from pinned host memory (H2D stream), runs forward+inverse
    # (compute stream) and reads the result back (D2H stream).  Two device
    # input buffers let step k+1's upload overlap step k's download (PCIe is
    # full duplex); stream events order each buffer's producer and consumer.
    xh = x.cpu().pin_memory()
    yh = [torch.empty_like(xh).pin_memory() for _ in range(2)]
    dev_in = [torch.empty_like(x) for _ in range(2)]
    comp = torch.cuda.current_stream()
    s_up, s_down = torch.cuda.Stream(), torch.cuda.Stream()
    loaded = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    computed = [torch.cuda.Event() for _ in range(2)]
    downloaded = [torch.cuda.Event() for _ in range(2)]
    for e in consumed + downloaded:
        e.record(comp)
    k_step = [0]

    def e2e_step():
        b = k_step[0] % 2
        k_step[0] += 1
        with torch.cuda.stream(s_up):
            s_up.wait_event(consumed[b])  # the compute of step k-2 has read dev_in[b]
            dev_in[b].copy_(xh, non_blocking=True)
            loaded[b].record(s_up)
        comp.wait_event(loaded[b])
        f = distfft.DistField(grid, distfft.Layout.Z_SLAB, distfft.Space.PHYSICAL, dev_in[b])
        spec = distfft.forward(f, w)
        consumed[b].record(comp)
        back = distfft.inverse(spec, w)
        computed[b].record(comp)
        with torch.cuda.stream(s_down):
            s_down.wait_event(computed[b])
            s_down.wait_event(downloaded[b])  # yh[b] of step k-2 is on the host
            yh[b].copy_(back.dev, non_blocking=True)
            back.dev.record_stream(s_down)
            downloaded[b].record(s_down)

    def drain():
        comp.wait_stream(s_up)
        comp.wait_stream(s_down)

    ms_e2e = timed(ctx, e2e_step, max(4, args.steps // 2), 2, drain=drain)
    torch.cuda.synchronize()
    e2e_err = float((yh[(k_step[0] - 1) % 2] - xh).norm() / xh.norm())
    bpr = fft_bytes(n)
    value = bpr / (ms * 1e-3) / 1e9
    out.update({
        "value": round(value, 2), "ms_per_step": round(ms, 4),
        "launches_total": launches,
        "e2e": {"value": round(bpr / (ms_e2e * 1e-3) / 1e9, 2), "unit": "GB/s",
                "ms_per_step": round(ms_e2e, 3),
                "h2d_bytes_per_step": int(ctx.sum_over_ranks(x.numel() * 8)),
                "d2h_bytes_per_step": int(ctx.sum_over_ranks(x.numel() * 8)),
                "pipeline": "H2D of step k+1 overlaps D2H of step k (separate copy streams)",
                "roundtrip_rel_l2": ctx.max_over_ranks(e2e_err)},
        "kernels": table,
        "parity": {"roundtrip_rel_l2": err, "tol": 1e-12, "ok": err <= 1e-12},
    })
    return table


def run_pfc2d(ctx, args):
    """configs[0]: 2D PFC 256^2, 100 semi-implicit steps (launch-bound; the
    single-rank path replays CUDA graphs), reference init and domain."""
    import torch

    from paper_2603_26818_b200 import distfft, pfc
    from paper_2603_26818_b200.grid import GridSpec, make_symbols

    n = (256, 256, 1)
    w = ctx.worker()
    grid = GridSpec(n, pfc.default_domain_length(n))
    psi0 = pfc.initial_field("constant_plus_noise", grid, psi_bar=-0.3, seed=0, noise_amplitude=0.01)
    f0 = distfft.scatter(psi0, w, grid, distfft.Layout.Y_SLAB, real=True)
    lay = distfft._layout(grid, distfft.Layout.X_SLAB, ctx.world, True)
    st = pfc.PfcState(psi_hat=distfft.forward(f0, w), grid=grid,
                      symbols=make_symbols(grid, -0.3, layout=lay, rank=ctx.rank), worker=w)
    params = pfc.PfcParams()
    pfc.pfc_run(st, params, 100)  # warm-up run (captures the graph)
    torch.cuda.synchronize()
    ctx.barrier()
    t0 = time.perf_counter()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    pfc.pfc_run(st, params, 100)
    b.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = ctx.max_over_ranks(a.elapsed_time(b) / 100)
    return {"metric": "PFC time-steps/sec", "value": round(1000.0 / ms, 1), "unit": "steps/s",
            "ms_per_step": round(ms, 5), "wall_s_per_100_steps": round(wall, 5),
            "config": "2D PFC 256x256 fp64 R2C, 100 steps (configs[0]), launch-bound"}


def run_multi(ctx, args):
    """configs[4]: multiphysics PFC (density + composition + 3 velocities),
    field-per-GPU: 1 GPU runs all roles, 4 GPUs the reference's four-role
    hydro dataflow, 5 / 8 GPUs the multiphysics role maps."""
    import numpy as np
    import torch

    from paper_2603_26818_b200 import hydro, multiphysics as mpx
    from paper_2603_26818_b200.grid import GridSpec, make_symbols
    from paper_2603_26818_b200.pfc import PfcParams

    G = ctx.world
    if G not in (1, 4, 5, 8):
        return None
    n = args.multi_n
    grid = GridSpec((n,) * 3, (2 * np.pi * np.sqrt(3) * (n // 8),) * 3)
    hp = hydro.HydroParams(pfc=PfcParams(eps=-0.3, dt=0.1), rho=1.0, gamma=1.0, a0=2.0)
    mp = mpx.MultiParams(hydro=hp, mobility=1.0, kappa=1.0, alpha=1.0, beta=0.0)
    sym = make_symbols(grid, -0.3, a0=2.0)
    gen = torch.Generator(device=ctx.device).manual_seed(11)
    C = torch.complex128

    def field(scale, base=0.0):
        x = torch.rand((n,) * 3, dtype=torch.float64, device=ctx.device, generator=gen)
        return (base + scale * (x - 0.5)).to(C)

    psi = field(0.02, -0.3)
    c = field(0.2)
    zeros = torch.zeros((n,) * 3, dtype=C, device=ctx.device)
    f = mpx.MultiFields(psi_hat=hydro._fft(psi, True), psi=psi, c_hat=hydro._fft(c, True), c=c,
                        v_hat=[zeros.clone() for _ in range(3)], v=[zeros.clone() for _ in range(3)])
    w = ctx.worker()
    torch.cuda.empty_cache()  # the FFT/PFC workloads' blocks are not reused here
    steps = max(3, args.steps // 4)
    if G == 1:
        fn = lambda: mpx.serial_multi_step(f, sym, mp)  # noqa: E731
        mode = "all 5 roles on 1 GPU"
    elif G == 4:
        hf = hydro.HydroFields(psi_hat=f.psi_hat, psi=f.psi, v_hat=f.v_hat, v=f.v)
        st = ({"psi_hat": hf.psi_hat, "psi": hf.psi, "v": list(hf.v), "step_index": 0} if ctx.rank == 0
              else {"v_hat": zeros.clone(), "psi": zeros.clone(), "step_index": 0})
        fn = lambda: hydro.parallel_hydro_step(w, st, sym, hp)  # noqa: E731
        mode = "reference 4-role hydro dataflow (psi, v1..v3), no composition"
    else:
        st = mpx.initial_role_state(ctx.rank, G, f)
        fn = lambda: mpx.parallel_multi_step(w, st, sym, mp)  # noqa: E731
        mode = f"{G}-role field-per-GPU map {mpx.ROLES[G]}"
    ms = timed(ctx, fn, steps, 2)
    return {"metric": "multiphysics PFC time-steps/sec", "value": round(1000.0 / ms, 3), "unit": "steps/s",
            "ms_per_step": round(ms, 3), "steps": steps,
            "config": f"{n}^3 complex128 full-grid fields, density+composition+v1..v3; {mode}"}


def run_pfc(ctx, args, n=None, steps=None, warmup=None):
    import torch

    from paper_2603_26818_b200 import _native as nat
    from paper_2603_26818_b200 import distfft, pfc
    from paper_2603_26818_b200.grid import GridSpec, make_symbols, slab_layout

    n = args.pfc_n if n is None else n
    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    w = ctx.worker()
    grid = GridSpec((n, n, n), pfc.default_domain_length((n, n, n)))
    cz = slab_layout(n, ctx.world).counts[ctx.rank]
    gen = torch.Generator(device=ctx.device).manual_seed(7 + ctx.rank)
    psi0 = torch.rand((n, n, cz), dtype=torch.float64, device=ctx.device, generator=gen)
    psi0.mul_(0.02).add_(-0.3 - 0.01)  # psi_bar - eta + 2 eta U(0,1)
    f0 = distfft.DistField(grid, distfft.Layout.Z_SLAB, distfft.Space.PHYSICAL, psi0)
    spec = distfft.forward(f0, w)
    del f0, psi0
    hl = distfft._layout(grid, distfft.Layout.X_SLAB, ctx.world, True)
    sym = make_symbols(grid, -0.3, layout=hl, rank=ctx.rank)
    st = pfc.PfcState(psi_hat=spec, grid=grid, symbols=sym, worker=w)
    params = pfc.PfcParams()
    mean0 = None
    if ctx.rank == 0:
        mean0 = float(st.psi_hat.dev.reshape(-1)[0].real.item())

    for _ in range(max(1, warmup)):
        pfc.pfc_run(st, params, 1)
    torch.cuda.synchronize()
    ctx.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    pfc.pfc_run(st, params, steps)  # K steps enqueued back to back, one read-back
    b.record()
    torch.cuda.synchronize()
    ctx.barrier()
    ms = ctx.max_over_ranks(a.elapsed_time(b) / steps)
    nat.trace = []
    pfc.pfc_run(st, params, max(2, steps // 4))
    torch.cuda.synchronize()
    table = kernel_table(nat.trace, max(2, steps // 4))
    nat.trace = None
    mass_ok = True
    if ctx.rank == 0:
        mass_ok = float(st.psi_hat.dev.reshape(-1)[0].real.item()) == mean0
    steps_s = 1000.0 / ms
    return {"metric": "PFC time-steps/sec", "value": round(steps_s, 3), "unit": "steps/s",
            "ms_per_step": round(ms, 4), "config": f"3D PFC {n}^3 fp64 R2C slab, dt=0.1 eps=-0.3",
            "kernels": table, "mass_bit_invariant": mass_ok,
            "alg_hbm_bytes_per_step": pfc_bytes(n) / ctx.world}


# ------------------------------------------------------------ CPU baseline --

def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_fft_baseline(n: int, seconds: float):
    """The reference's slab-decomposed C2C round trip (distfft.py:150-173 on
    transport.py's thread group) restated in oracle/ref_numpy.py, with one
    worker thread per host core; repeated until `seconds` of work."""
    import numpy as np

    sys.path.insert(0, str(ROOT / "oracle"))
    import ref_numpy as ora

    cores = cpu_cores()
    x = np.random.default_rng(0).standard_normal((n, n, n))
    times = []
    t_end = time.perf_counter() + seconds
    while True:
        t0 = time.perf_counter()
        _, back = ora.dist_roundtrip_threads(x, cores)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end or len(times) >= 10:
            break
    best = min(times)
    return {"value": round(fft_bytes(n) / best / 1e9, 4), "unit": "GB/s", "cores": cores,
            "kind": "port", "s_per_roundtrip": round(best, 3),
            "sample": f"{len(times)} x C2C round trip of a real {n}^3 fp64 field (reference "
                      f"algorithm, {cores} worker threads), best of {len(times)}"}


def main():
    args = parse()
    hbm, peak_kind = peaks()
    if args.impl == "reference":
        return main_reference(args)
    ctx = Ctx(args.gpus)
    out = {"metric": "distributed 3D FFT GB/s (fp64)", "unit": "GB/s", "n_gpus": ctx.world,
           "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"3D R2C/C2R FFT round trip {args.fft_n}^3 fp64 (forward + inverse, "
                                  f"slab decomposition)",
                      "grid": [args.fft_n] * 3, "decomposition": f"slab x{ctx.world}",
                      "l2": "inputs (1 GiB per field at 512^3) exceed the 126 MB L2; no flush needed"}}
    with ClockSampler(ctx.device.index) as clk:
        table = run_fft(ctx, args, out)
        pfc_res = None if args.no_pfc else run_pfc(ctx, args)
        # configs[3] grid (2048^3) when it is comfortably in this run's reach:
        # at N >= 4 GPUs (slab, <= ~70 GB peak per rank incl. the exchange
        # buffers) or with --pfc-big on one GPU (R2C state 2 x 68.8 GB); a
        # failure is reported, not fatal
        pfc_big = None
        if not args.no_pfc and (ctx.world >= 4 or args.pfc_big):
            import torch

            pfc_res_keep = pfc_res
            torch.cuda.empty_cache()
            try:
                pfc_big = run_pfc(ctx, args, n=args.pfc_big_n, steps=max(3, args.steps // 4), warmup=2)
            except Exception as exc:  # noqa: BLE001 - keep the rest of the line
                pfc_big = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
            torch.cuda.empty_cache()
            pfc_res = pfc_res_keep
        pfc2d = None if args.no_pfc else run_pfc2d(ctx, args)
        multi = None if args.no_multi else run_multi(ctx, args)
    out["clocks"] = clk.summary()
    workload = f"fft{args.fft_n}" if ctx.world == 1 else None
    out["roofline"] = roofline_of(table, hbm, peak_kind, measured_traffic(workload))
    out["roofline"]["whole_step_frac"] = round(out["value"] / (hbm * ctx.world), 4)
    if pfc_res is not None:
        pr = roofline_of(pfc_res["kernels"], hbm, peak_kind,
                         measured_traffic(f"pfc{args.pfc_n}") if ctx.world == 1 else None)
        pfc_res["roofline"] = pr
        t_roof = pfc_res["alg_hbm_bytes_per_step"] / (hbm * 1e9)
        pfc_res["roofline_step_frac"] = round(t_roof / (pfc_res["ms_per_step"] * 1e-3), 4)
        out["pfc"] = pfc_res
    if pfc_big is not None:
        if "error" not in pfc_big:
            t_roof = pfc_big["alg_hbm_bytes_per_step"] / (hbm * 1e9)
            pfc_big["roofline_step_frac"] = round(t_roof / (pfc_big["ms_per_step"] * 1e-3), 4)
            pfc_big["config"] += " (configs[3] grid; slab decomposition)" if args.pfc_big_n == 2048 else ""
        out["pfc2048"] = pfc_big
    if pfc2d is not None:
        out["pfc2d"] = pfc2d
    if multi is not None:
        out["multiphysics"] = multi
    out["gpu_launches"] = int(out.pop("launches_total"))
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_fft_baseline(args.fft_n, args.cpu_seconds)
    if ctx.rank == 0:
        print(json.dumps(out))
    if ctx.dist is not None:
        ctx.dist.destroy_process_group()


def main_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import numpy as np

    sys.path.insert(0, str(ROOT / "oracle"))
    import ref_numpy as ora

    n = args.fft_n
    cores = cpu_cores()
    x = np.random.default_rng(0).standard_normal((n, n, n))
    for _ in range(max(0, min(args.warmup, 1))):
        ora.dist_roundtrip_threads(x, cores)
    times = []
    budget = time.perf_counter() + 150.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ora.dist_roundtrip_threads(x, cores)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > budget:
            break
    s = sum(times) / len(times)
    v = fft_bytes(n) / s / 1e9
    out = {"impl": "reference", "metric": "distributed 3D FFT GB/s (fp64)", "value": round(v, 4),
           "unit": "GB/s", "n_gpus": world, "steps": len(times), "warmup": args.warmup,
           "ms_per_step": round(s * 1e3, 2), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"3D FFT round trip {n}^3 fp64 (reference C2C slab algorithm on "
                                  f"host threads)", "grid": [n] * 3},
           "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": cores, "kind": "port",
                            "sample": f"{len(times)} C2C round trips of a real {n}^3 field, "
                                      f"{cores} worker threads (oracle restatement of distfft.py)"},
           "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
