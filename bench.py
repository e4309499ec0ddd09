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
    ap.add_argument("--no-cpu-sub", action="store_true", help="skip the sub-lines' CPU baselines")
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


KERNELS_NOTE = ("per-kernel times from a separate traced pass of the same steps (CUDA events recorded on the "
                "launching stream around every launch); the tracing serialises launches, so the kernels sum to "
                "a few % more than the untraced ms_per_step")


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

    # >= 48 steps: the timed region starts and ends with empty copy queues, so
    # one upload and one download (~21 ms each at 512^3) are not overlapped;
    # over K steps that fill/drain costs ~1/K of the rate (24 steps: 4 %)
    ms_e2e = timed(ctx, e2e_step, max(48, args.steps), 2, drain=drain)
    torch.cuda.synchronize()
    e2e_err = float((yh[(k_step[0] - 1) % 2] - xh).norm() / xh.norm())

    # the same copy pipeline with no compute: the PCIe bound of the e2e step
    def copy_step():
        b = k_step[0] % 2
        k_step[0] += 1
        with torch.cuda.stream(s_up):
            s_up.wait_event(downloaded[b])
            dev_in[b].copy_(xh, non_blocking=True)
            loaded[b].record(s_up)
        with torch.cuda.stream(s_down):
            s_down.wait_event(loaded[b])
            yh[b].copy_(dev_in[b], non_blocking=True)
            downloaded[b].record(s_down)

    ms_copy = timed(ctx, copy_step, max(48, args.steps), 2, drain=drain)
    torch.cuda.synchronize()
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
                "copy_only_ms_per_step": round(ms_copy, 3),
                "pcie_gbs_per_direction": round(x.numel() * 8 / (ms_copy * 1e-3) / 1e9, 2),
                "frac_of_copy_bound": round(ms_copy / ms_e2e, 4),
                "roundtrip_rel_l2": ctx.max_over_ranks(e2e_err)},
        "kernels": table,
        "kernels_note": KERNELS_NOTE,
        "parity": {"roundtrip_rel_l2": err, "tol": 1e-12, "ok": err <= 1e-12},
    })
    return table


def pfc_e2e(ctx, st, params, phys_layout, host_in, steps: int) -> dict:
    """The PFC metric end to end through the public API with host buffers:
    pinned host psi -> H2D -> distfft.forward -> (into the state) ->
    pfc.pfc_run(steps) (diagnostics read back) -> distfft.inverse -> D2H,
    everything inside the CUDA-event timed region.  One warm-up run first;
    steps/s = steps / time, copies counted per step."""
    import torch

    from paper_2603_26818_b200 import distfft, pfc

    w = st.worker
    dev_in = torch.empty(host_in.shape, dtype=host_in.dtype, device=ctx.device)
    host_out = torch.empty_like(host_in).pin_memory()
    diag_bytes = 64 * 4 * 8 * steps  # the per-step diagnostics block pfc_run reads back

    def once():
        dev_in.copy_(host_in, non_blocking=True)
        f = distfft.DistField(st.grid, phys_layout, distfft.Space.PHYSICAL, dev_in)
        spec = distfft.forward(f, w)
        st.psi_hat.dev.copy_(spec.dev)
        st.psi_hat.touch()
        del spec
        pfc.pfc_run(st, params, steps)
        back = distfft.inverse(st.psi_hat, w)
        host_out.copy_(back.dev, non_blocking=True)

    once()
    torch.cuda.synchronize()
    ctx.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    once()
    b.record()
    torch.cuda.synchronize()
    ms = ctx.max_over_ranks(a.elapsed_time(b))
    nb = host_in.numel() * host_in.element_size()
    return {"value": round(1000.0 * steps / ms, 3), "unit": "steps/s", "ms_per_run": round(ms, 3),
            "steps_per_run": steps,
            "h2d_bytes_per_step": int(ctx.sum_over_ranks(nb) / steps),
            "d2h_bytes_per_step": int(ctx.sum_over_ranks(nb + diag_bytes) / steps),
            "pipeline": f"host psi in (pinned) -> forward -> pfc_run({steps}) -> inverse -> host psi out; "
                        f"copies amortised over the run's steps"}


def run_pfc2d(ctx, args):
    """configs[0]: 2D PFC 256^2, 100 semi-implicit steps (launch-bound; the
    single-rank path replays CUDA graphs), reference init and domain."""
    import numpy as np
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
    host = torch.from_numpy(np.array(f0.local)).pin_memory()
    e2e = pfc_e2e(ctx, st, params, distfft.Layout.Y_SLAB, host, 100)
    return {"metric": "PFC time-steps/sec", "value": round(1000.0 / ms, 1), "unit": "steps/s",
            "ms_per_step": round(ms, 5), "wall_s_per_100_steps": round(wall, 5),
            "config": "2D PFC 256x256 fp64 R2C, 100 steps (configs[0]), launch-bound", "e2e": e2e}


def multi_bytes(n: int) -> float:
    """Algorithmic HBM bytes of one serial R2C multiphysics step (beta = 0),
    R = 8 n^3 (a real field), S = spec_bytes(n) (a half spectrum), as the
    fused schedule moves them:
      * 23 transforms of R + 5S (R + S for the x pass, 2S for y and z each)
        = 23R + 115S;
      * the real pointwise work of the unfused schedule, 17R: the two
        v . grad x products (6 reads + 1 write each: 14R) and the second
        factor psi of the three forces (3R);
      * less what the fused x passes keep out of HBM: each force
        (pfcs_xmul_x: C2R, * psi, R2C in one pass) the derivative's write
        and re-read (3 x -2R), each advection (pfcs_xdot3_x: three C2R, the
        dot product, the R2C in one pass) the three derivatives' writes and
        re-reads, the product's write and re-read (2 x -8R: its 3R of
        velocity reads remain);
      * the spectral updates / mu: psi 4S, c 4S, mu 3S, 3 x velocity 3S = 20S,
        less the five state updates' re-read of the new state (they ride in
        the z pass of their inverse, pfcs_update_zinv: -5S);
      * one z pass (2S) less per gradient (grad psi, grad c, grad mu: the x
        and y derivatives share one inverse z pass, _Real3.grad_inv: -6S);
      * mu fused with its two operands' forward z passes (pfcs_hydro_mu_z:
        2S read, S written instead of the two z passes' 4S and the mu
        pass's 3S: -4S);
      * the density update's F(psi^3) carried over from the previous step's
        mu (same psi: one forward transform, R + 5S, less per step; the
        fused mu kernel writes it, +S: -R - 4S);
      * the shared inverse z pass of grad psi and grad c carried over from
        the psi and c updates (their fused z pass already computed it; the
        y pass that follows runs out of place to keep it: -2 x 2S);
      * the updates take their operands before the forward z pass and run
        it in registers (pfcs_update_zzinv: each such operand's z-pass
        write and re-read, 2S — psi: adv; c: f and adv; v_1..3: the force:
        -12S);
      * grad mu's first inverse z passes run inside the mu kernel
        (pfcs_hydro_mu_zgrad: mu_hat is never stored nor re-read by the
        two z passes: -3S);
      * the x derivative of grad psi / grad c takes its i k_x in the
        advection x pass (pfcs_xdot3_x dx), so it starts from the update's
        kept y pass instead of a y pass of its own (-2 x 2S).
    Total 17R + 93S."""
    R = 8.0 * n**3
    S = spec_bytes(n)
    return 23 * (R + 5 * S) + (17 - 6 - 16 - 1) * R + (20 - 5 - 6 - 4 - 4 - 4 - 12 - 3 - 4) * S


def run_multi(ctx, args):
    """configs[4]: multiphysics PFC (density + composition + 3 velocities),
    field-per-GPU: 1 GPU runs all roles, 5 / 8 GPUs the multiphysics role
    maps, 4 GPUs the reference's four-role hydro dataflow — all on real
    fields (the R2C path)."""
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

    def field(scale, base=0.0):  # real physical fields: every role map takes the R2C path
        x = torch.rand((n,) * 3, dtype=torch.float64, device=ctx.device, generator=gen)
        return base + scale * (x - 0.5)

    psi = field(0.02, -0.3)
    c = field(0.2)
    w = ctx.worker()
    R3 = mpx._Real3.of((n,) * 3, sym, ctx.device)
    zeros = torch.zeros((n,) * 3, dtype=torch.float64, device=ctx.device)
    f = mpx.MultiFields(psi_hat=R3.fwd(psi), psi=psi, c_hat=R3.fwd(c), c=c,
                        v_hat=[R3.fwd(zeros) for _ in range(3)], v=[zeros.clone() for _ in range(3)])
    torch.cuda.empty_cache()  # the FFT/PFC workloads' blocks are not reused here
    steps = max(3, args.steps // 4)
    if G == 1:
        fn = lambda: mpx.serial_multi_step(f, sym, mp)  # noqa: E731
        mode = "all 5 roles on 1 GPU (R2C: real fields, x-halved spectra)"
    elif G == 4:
        st = ({"psi_hat": f.psi_hat, "psi": f.psi, "v": list(f.v), "step_index": 0} if ctx.rank == 0
              else {"v_hat": f.v_hat[ctx.rank - 1].clone(), "psi": zeros.clone(), "step_index": 0})
        fn = lambda: hydro.parallel_hydro_step(w, st, sym, hp)  # noqa: E731
        mode = "reference 4-role hydro dataflow (psi, v1..v3; R2C), no composition"
    else:
        st = mpx.initial_role_state(ctx.rank, G, f)
        fn = lambda: mpx.parallel_multi_step(w, st, sym, mp)  # noqa: E731
        mode = f"{G}-role field-per-GPU map {mpx.ROLES[G]} (R2C)"
    ms = timed(ctx, fn, steps, 2)
    res = {"metric": "multiphysics PFC time-steps/sec", "value": round(1000.0 / ms, 3), "unit": "steps/s",
           "ms_per_step": round(ms, 3), "steps": steps,
           "config": f"{n}^3 fp64 density+composition+v1..v3; {mode}"}
    if G == 1:
        hbm, kind = peaks()
        alg = multi_bytes(n)
        res["roofline"] = {"bound": "hbm", "alg_bytes_per_step": alg, "achieved": round(alg / (ms * 1e-3) / 1e9, 1),
                           "peak": hbm, "unit": "GB/s", "frac": round(alg / (ms * 1e-3) / 1e9 / hbm, 4),
                           "model": "fused schedule, 17R + 93S per step (R a real field, S a half spectrum; "
                                    "pass-by-pass in bench.multi_bytes)"}
        # e2e: host psi, c (pinned) in -> forward transforms -> K steps -> psi, c, v out
        hp_in = [x.cpu().pin_memory() for x in (psi, c)]
        outs = [torch.empty_like(hp_in[0]).pin_memory() for _ in range(5)]

        def run_e2e():
            dev = [x.to(ctx.device, non_blocking=True) for x in hp_in]
            z = torch.zeros_like(dev[0])
            ff = mpx.MultiFields(psi_hat=R3.fwd(dev[0]), psi=dev[0], c_hat=R3.fwd(dev[1]), c=dev[1],
                                 v_hat=[R3.fwd(z) for _ in range(3)], v=[z.clone() for _ in range(3)])
            for _ in range(steps):
                mpx.serial_multi_step(ff, sym, mp)
            for o, x in zip(outs, [ff.psi, ff.c, *ff.v]):
                o.copy_(x, non_blocking=True)

        run_e2e()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        run_e2e()
        b.record()
        torch.cuda.synchronize()
        ms_e = a.elapsed_time(b)
        nb = hp_in[0].numel() * 8
        res["e2e"] = {"value": round(1000.0 * steps / ms_e, 3), "unit": "steps/s", "ms_per_run": round(ms_e, 3),
                      "steps_per_run": steps, "h2d_bytes_per_step": int(2 * nb / steps),
                      "d2h_bytes_per_step": int(5 * nb / steps),
                      "pipeline": f"host psi, c in (pinned) -> forward transforms -> {steps} serial steps -> host "
                                  f"psi, c, v1..v3 out; per-step divergence flag read back"}
    return res


def run_pfc(ctx, args, n=None, steps=None, warmup=None, e2e=True):
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
    host = psi0.cpu().pin_memory() if e2e else None
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
    res = {"metric": "PFC time-steps/sec", "value": round(steps_s, 3), "unit": "steps/s",
           "ms_per_step": round(ms, 4), "config": f"3D PFC {n}^3 fp64 R2C slab, dt=0.1 eps=-0.3",
           "kernels": table, "kernels_note": KERNELS_NOTE, "mass_bit_invariant": mass_ok,
           "alg_hbm_bytes_per_step": pfc_bytes(n) / ctx.world}
    if e2e:
        res["e2e"] = pfc_e2e(ctx, st, params, distfft.Layout.Z_SLAB, host, steps)
    return res


def run_pfc_pencil(ctx, args, n: int, steps: int, warmup: int = 2) -> dict:
    """configs[3]: 3D PFC on a pr x pc pencil grid (PencilGrid.for_workers(G):
    2 x 4 at G = 8) — x-pencil physical field, z-pencil half spectrum, row
    and column all-to-alls (pencil.py), same timing rules as run_pfc."""
    import torch

    from paper_2603_26818_b200 import distfft, pfc
    from paper_2603_26818_b200.grid import GridSpec, make_symbols
    from paper_2603_26818_b200.pencil import PencilGeometry, PencilGrid, PencilLayout

    pg = PencilGrid.for_workers(ctx.world)
    w = ctx.worker()
    grid = GridSpec((n, n, n), pfc.default_domain_length((n, n, n)))
    g = PencilGeometry(grid, pg, ctx.rank, True)
    gen = torch.Generator(device=ctx.device).manual_seed(17 + ctx.rank)
    x = torch.rand((n, g.cy, g.cz), dtype=torch.float64, device=ctx.device, generator=gen)
    x.mul_(0.02).add_(-0.31)
    f0 = distfft.DistField(grid, PencilLayout(pg, "x"), distfft.Space.PHYSICAL, x)
    st = pfc.PfcState(psi_hat=distfft.forward(f0, w), grid=grid, symbols=make_symbols(grid, -0.3), worker=w)
    del f0, x
    params = pfc.PfcParams()
    for _ in range(max(1, warmup)):
        pfc.pfc_run(st, params, 1)
    torch.cuda.synchronize()
    ctx.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    pfc.pfc_run(st, params, steps)
    b.record()
    torch.cuda.synchronize()
    ctx.barrier()
    ms = ctx.max_over_ranks(a.elapsed_time(b) / steps)
    hbm, _ = peaks()
    res = {"metric": "PFC time-steps/sec", "value": round(1000.0 / ms, 3), "unit": "steps/s",
           "ms_per_step": round(ms, 4), "steps": steps,
           "config": f"3D PFC {n}^3 fp64 R2C pencil {pg.pr}x{pg.pc} (configs[3] decomposition)",
           "alg_hbm_bytes_per_step": pfc_bytes(n) / ctx.world}
    # each rank moves its half-spectrum share twice through the row and twice
    # through the column all-to-all per step
    S = spec_bytes(n)
    nv = 2 * S / ctx.world * ((pg.pr - 1) / pg.pr + (pg.pc - 1) / pg.pc)
    t_hbm = pfc_bytes(n) / (ctx.world * hbm * 1e9)
    t_nvl = nv / (NVLINK_GBS * 1e9)
    res["roofline_combined"] = {"t_roof_ms": round(1e3 * (t_hbm + t_nvl), 4), "t_hbm_ms": round(1e3 * t_hbm, 4),
                                "t_nvlink_ms": round(1e3 * t_nvl, 4), "nvlink_bytes_per_gpu": nv,
                                "frac": round((t_hbm + t_nvl) / (ms * 1e-3), 4)}
    return res


# ------------------------------------------------------------ CPU baseline --
# The reference's CPU path, timed on this box's host cores.  Preferred: the
# UNMODIFIED reference package staged by oracle/vendor_reference.py under
# oracle/_ref/pfcspectral (kind "reference"); where it was not staged, the
# oracle's restatement (kind "port").  Sizes the reference cannot hold in host
# RAM (1024^3: ~210 B/point) use the oracle's lean R2C restatement, labelled.

def cpu_info() -> dict:
    try:
        import psutil

        phys, logical = psutil.cpu_count(logical=False), psutil.cpu_count()
    except Exception:
        phys, logical = None, os.cpu_count()
    model = None
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = logical
    return {"physical_cores": phys, "logical_cpus": logical, "usable_cpus": usable, "model": model}


def cpu_threads() -> int:
    """Worker threads for the CPU reference: every usable logical CPU (numpy's
    pocketfft releases the GIL, so the reference's thread workers scale)."""
    return cpu_info()["usable_cpus"] or 1


def host_gib() -> float:
    try:
        import psutil

        return psutil.virtual_memory().available / 2**30
    except Exception:
        return 0.0


def ref_package():
    """The unmodified reference package (oracle/_ref/pfcspectral), or None."""
    d = ROOT / "oracle" / "_ref"
    if not (d / "pfcspectral" / "__init__.py").exists():
        return None
    if str(d) not in sys.path:
        sys.path.insert(0, str(d))
    import pfcspectral

    return pfcspectral


def _oracle():
    sys.path.insert(0, str(ROOT / "oracle"))
    import ref_numpy

    return ref_numpy


def ref_fft_roundtrips(n: int, threads: int, steps: int, budget_s: float):
    """distfft.forward + inverse (distfft.py:150-173) of a real n^3 field over
    spawn_group(threads) (transport.py:174-200), each round trip bracketed by
    worker barriers; returns (seconds per round trip list, kind)."""
    import numpy as np

    x = np.random.default_rng(0).standard_normal((n, n, n))
    ref = ref_package()
    if ref is None:
        ora = _oracle()
        ora.dist_roundtrip_threads(x, threads)  # warm-up
        times = []
        t_end = time.perf_counter() + budget_s
        for _ in range(steps):
            t0 = time.perf_counter()
            ora.dist_roundtrip_threads(x, threads)
            times.append(time.perf_counter() - t0)
            if time.perf_counter() > t_end:
                break
        return times, "port"
    from pfcspectral import distfft as rdf
    from pfcspectral.grid import GridSpec as RGrid
    from pfcspectral.transport import spawn_group as rspawn

    grid = RGrid((n, n, n), (1.0, 1.0, 1.0))
    plan = {"steps": steps}

    def body(w):
        f = rdf.scatter(x, w, grid, rdf.Layout.Z_SLAB)
        w.barrier()
        t0 = time.perf_counter()
        rdf.inverse(rdf.forward(f, w), w)  # warm-up round trip, sizes the sample
        w.barrier()
        t1 = time.perf_counter() - t0
        if w.rank == 0:
            plan["steps"] = max(1, min(steps, int(budget_s / max(t1, 1e-9))))
        w.barrier()
        out = []
        for _ in range(plan["steps"]):
            t0 = time.perf_counter()
            rdf.inverse(rdf.forward(f, w), w)
            w.barrier()
            out.append(time.perf_counter() - t0)
        return out

    return rspawn(threads, body, timeout=600.0)[0], "reference"


def cpu_fft_baseline(n: int, seconds: float) -> dict:
    threads = cpu_threads()
    times, kind = ref_fft_roundtrips(n, threads, 10, seconds)
    best = min(times)
    src = ("reference package pfcspectral (oracle/_ref), distfft.forward/inverse over spawn_group"
           if kind == "reference" else "oracle restatement of distfft.py on host threads")
    return {"value": round(fft_bytes(n) / best / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": kind,
            "s_per_roundtrip": round(best, 3), "host": cpu_info(),
            "sample": f"{len(times)} C2C round trips of a real {n}^3 fp64 field ({src}, {threads} worker "
                      f"threads), best of {len(times)}"}


def cpu_pfc2d_baseline(steps: int = 100) -> dict | None:
    """configs[0] on the host: the reference's pfc_step (pfc.py:96-128) on 2D
    256^2, 100 steps, G = 1 and G = 4 thread workers (its fastest count in
    SURVEY.md §6); reports the faster."""
    ref = ref_package()
    if ref is None:
        return None
    from pfcspectral import distfft as rdf, pfc as rpfc
    from pfcspectral.grid import GridSpec as RGrid, make_symbols as rsym
    from pfcspectral.transport import spawn_group as rspawn

    n = (256, 256, 1)
    grid = RGrid(n, rpfc.default_domain_length(n))
    psi0 = rpfc.initial_field("constant_plus_noise", grid, psi_bar=-0.3, seed=0, noise_amplitude=0.01)
    params = rpfc.PfcParams()
    best = None
    for G in sorted({1, min(4, cpu_threads())}):
        def body(w):
            lay = rdf.layout_for(grid, rdf.Layout.X_SLAB, w.size)
            st = rpfc.PfcState(psi_hat=rdf.forward(rdf.scatter(psi0, w, grid, rdf.physical_layout(grid)), w),
                               grid=grid, symbols=rsym(grid, -0.3, layout=lay, rank=w.rank), worker=w)
            w.barrier()
            t0 = time.perf_counter()
            for _ in range(steps):
                rpfc.pfc_step(st, params)
            w.barrier()
            return time.perf_counter() - t0

        t = max(rspawn(G, body, timeout=600.0)) / steps
        if best is None or t < best[0]:
            best = (t, G)
    return {"value": round(1.0 / best[0], 2), "unit": "steps/s", "cores": best[1], "kind": "reference",
            "sample": f"{steps} steps of the reference pfc_step on 2D 256^2 (configs[0]), best of G = 1 / "
                      f"{min(4, cpu_threads())} thread workers (G = {best[1]} fastest)"}


def cpu_pfc3d_baseline(n: int) -> dict | None:
    """configs[2] grid on the host: the reference itself needs ~210 B/point of
    RAM (~210 GiB at 1024^3), so one step of the oracle's lean R2C
    restatement of pfc.py:96-128 (scipy pocketfft, all host threads) is timed
    instead, labelled as such; at 512^3 when the host lacks the RAM for n."""
    import numpy as np

    ora = _oracle()
    threads = cpu_threads()
    m = n
    while m > 256 and host_gib() < 48.0 * (m / 1024) ** 3 + 4:
        m //= 2
    shape = (m, m, m)
    psi_hat = np.fft.rfftn(-0.3 + np.random.default_rng(0).uniform(-0.01, 0.01, shape), axes=(1, 2, 0))
    L = (2 * np.pi * np.sqrt(3) * (m // 8),) * 3
    ora.pfc_step_r2c_lean(np.zeros((5, 8, 8), np.complex128), (8, 8, 8), L, -0.3, 0.1, workers=threads)  # warm-up
    t0 = time.perf_counter()
    ora.pfc_step_r2c_lean(psi_hat, shape, L, -0.3, 0.1, workers=threads)
    t = time.perf_counter() - t0
    return {"value": round(1.0 / t, 5), "unit": "steps/s", "cores": threads, "kind": "port",
            "grid": list(shape), "s_per_step": round(t, 3),
            "sample": f"1 step of the oracle's lean R2C restatement of pfc.pfc_step at {m}^3 (the reference "
                      f"package needs ~210 B/point of host RAM: not runnable at {n}^3), scipy pocketfft with "
                      f"{threads} threads"}


def cpu_hydro_baseline(n: int = 128) -> dict | None:
    """configs[4] on the host, scaled down: the reference's serial 4-field
    hydro step (hydro.py:110-126) at 128^3 (512^3 needs ~40 GiB and minutes
    per step); the composition field has no reference."""
    import numpy as np

    ref = ref_package()
    if ref is None:
        return None
    from pfcspectral import hydro as rh
    from pfcspectral.fftcore import fft_nd as rfft
    from pfcspectral.grid import GridSpec as RGrid, make_symbols as rsym
    from pfcspectral.pfc import PfcParams as RP

    grid = RGrid((n,) * 3, (2 * np.pi * np.sqrt(3) * (n // 8),) * 3)
    sym = rsym(grid, -0.3, a0=2.0)
    hp = rh.HydroParams(pfc=RP(eps=-0.3, dt=0.1), rho=1.0, gamma=1.0, a0=2.0)
    psi = (-0.3 + 0.02 * (np.random.default_rng(11).random((n,) * 3) - 0.5)).astype(np.complex128)
    z = np.zeros((n,) * 3, np.complex128)
    f = rh.HydroFields(psi_hat=rfft(psi), psi=psi, v_hat=[z.copy() for _ in range(3)], v=[z.copy() for _ in range(3)])
    rh.serial_hydro_step(f, sym, hp)
    t0 = time.perf_counter()
    rh.serial_hydro_step(f, sym, hp)
    t = time.perf_counter() - t0
    return {"value": round(1.0 / t, 4), "unit": "steps/s", "cores": 1, "kind": "reference",
            "grid": [n] * 3, "s_per_step": round(t, 3),
            "sample": f"1 serial 4-field hydro step (psi, v1..v3) of the reference package at {n}^3 on one "
                      f"thread (serial mode; 512^3 is out of the few-minute budget)"}


def spec_bytes(n: int) -> float:
    """S: one R2C half spectrum of an n^3 fp64 field."""
    return 16.0 * n * n * (n // 2 + 1)


NVLINK_GBS = 770.0  # measured peer copy per direction per GPU (B200_PROFILING.md); nominal 900


def combined_roofline(hbm_bytes: float, xchg_bytes: float, G: int, hbm_gbs: float, ms: float) -> dict:
    """t_roof = HBM bytes / (G B_HBM) + each GPU's transpose bytes
    X (G-1)/G^2 / B_NVL (SURVEY.md §8d phase-sum); frac = t_roof / t."""
    t_hbm = hbm_bytes / (G * hbm_gbs * 1e9)
    nv = xchg_bytes * (G - 1) / (G * G)
    t_nvl = nv / (NVLINK_GBS * 1e9)
    t_nom = hbm_bytes / (G * hbm_gbs * 1e9) + nv / 900e9
    return {"t_roof_ms": round(1e3 * (t_hbm + t_nvl), 4), "t_hbm_ms": round(1e3 * t_hbm, 4),
            "t_nvlink_ms": round(1e3 * t_nvl, 4), "nvlink_bytes_per_gpu": nv,
            "frac": round((t_hbm + t_nvl) / (ms * 1e-3), 4), "frac_nominal_nvlink_900": round(t_nom / (ms * 1e-3), 4),
            "peaks": {"hbm_gbs": hbm_gbs, "nvlink_gbs": NVLINK_GBS}}


def _guard(fn):
    try:
        return fn()
    except Exception as exc:  # noqa: BLE001 - a failed side measurement is reported, not fatal
        return {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}


def run_yardstick(ctx, args) -> dict:
    """Non-product yardstick: cuFFT (torch.fft.rfftn / irfftn, fp64) on the
    same 512^3 round trip, same algorithmic bytes, CUDA events."""
    import torch

    n = args.fft_n
    x = torch.randn((n, n, n), dtype=torch.float64, device=ctx.device)

    def step():
        torch.fft.irfftn(torch.fft.rfftn(x), s=(n, n, n))

    ms = timed(ctx, step, max(5, args.steps // 2), 3)
    del x
    torch.cuda.empty_cache()
    return {"impl": "cuFFT via torch.fft.rfftn/irfftn (library, not the product path)",
            "ms_per_step": round(ms, 4), "value": round(fft_bytes(n) / (ms * 1e-3) / 1e9, 1), "unit": "GB/s"}


def run_exchange(ctx, args) -> dict:
    """N > 1: the 1024^3 R2C transpose alone as NCCL all_to_all_single (bus
    GB/s = bytes each rank sends to the others / time, nccl-tests
    all-to-all convention) vs NVLink's 770 GB/s measured / 900 nominal."""
    import torch

    from paper_2603_26818_b200.grid import slab_layout

    if ctx.dist.get_backend() != "nccl":
        return {"skipped": "NCCL all-to-all microbenchmark needs the nccl backend (gloo smoke run)"}
    n, G = args.pfc_n, ctx.world
    nxm = n // 2 + 1
    xl, zl = slab_layout(nxm, G), slab_layout(n, G)
    me = ctx.rank
    # Z slab -> X slab: my (nxm, n, cz_me) block rows xl[h] go to rank h
    send_counts = [xl.counts[h] * n * zl.counts[me] for h in range(G)]
    recv_counts = [xl.counts[me] * n * zl.counts[h] for h in range(G)]
    send = torch.randn(sum(send_counts), dtype=torch.complex128, device=ctx.device)
    recv = torch.empty(sum(recv_counts), dtype=torch.complex128, device=ctx.device)

    def step():
        ctx.dist.all_to_all_single(recv, send, output_split_sizes=recv_counts, input_split_sizes=send_counts)

    ms = timed(ctx, step, 10, 3)
    off = (sum(send_counts) - send_counts[me]) * 16
    bus = ctx.max_over_ranks(off) / (ms * 1e-3) / 1e9
    del send, recv
    torch.cuda.empty_cache()
    return {"nccl_all_to_all": {"grid": [n] * 3, "ms": round(ms, 4), "bytes_to_peers_per_rank": off,
                                "bus_gbs": round(bus, 1), "frac_of_770": round(bus / NVLINK_GBS, 4),
                                "frac_of_900": round(bus / 900.0, 4)},
            "note": "the PFC step's default transposes are fused into the FFT kernels' stores "
                    "(pfc kernels fft_lines_scatter / pfc_update_z_to); their time is in pfc.kernels"}


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
        # (before the PFC lines: after a 137 GB 2048^3 run the 512^3
        # multiphysics step measured 41 instead of 27 ms on the same box,
        # after the 1024^3 line 28.6)
        multi = None if args.no_multi else run_multi(ctx, args)
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
                pfc_big = run_pfc(ctx, args, n=args.pfc_big_n, steps=max(3, args.steps // 4), warmup=2, e2e=False)
            except Exception as exc:  # noqa: BLE001 - keep the rest of the line
                pfc_big = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
            torch.cuda.empty_cache()
            pfc_res = pfc_res_keep
        pencil = None
        if not args.no_pfc and ctx.world >= 4:
            import torch

            torch.cuda.empty_cache()
            pencil = _guard(lambda: run_pfc_pencil(ctx, args, args.pfc_big_n, max(3, args.steps // 4)))
            torch.cuda.empty_cache()
        pfc2d = None if args.no_pfc else run_pfc2d(ctx, args)
        exch = run_exchange(ctx, args) if ctx.world > 1 and not args.no_pfc else None
        yard = _guard(lambda: run_yardstick(ctx, args)) if ctx.world == 1 else None
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
    if pencil is not None:
        out["pfc_pencil"] = pencil
    if pfc2d is not None:
        out["pfc2d"] = pfc2d
    if multi is not None:
        out["multiphysics"] = multi
    # combined HBM + NVLink roofline: phase-sum of the HBM
    # passes over G GPUs and each GPU's share of the transposes over NVLink
    G = ctx.world
    out["roofline"]["combined"] = combined_roofline(fft_bytes(args.fft_n), 2 * spec_bytes(args.fft_n), G, hbm,
                                                    out["ms_per_step"])
    if pfc_res is not None:
        pfc_res["roofline"]["combined"] = combined_roofline(pfc_bytes(args.pfc_n), 2 * spec_bytes(args.pfc_n), G,
                                                            hbm, pfc_res["ms_per_step"])
    if pfc_big is not None and "error" not in pfc_big:
        pfc_big["roofline_combined"] = combined_roofline(pfc_bytes(args.pfc_big_n), 2 * spec_bytes(args.pfc_big_n),
                                                         G, hbm, pfc_big["ms_per_step"])
    if exch is not None:
        out["exchange"] = exch
    if yard is not None:
        out["yardstick"] = yard
    out["gpu_launches"] = int(out.pop("launches_total"))
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_fft_baseline(args.fft_n, args.cpu_seconds)
        if not args.no_cpu_sub:
            if pfc_res is not None:
                pfc_res["cpu_baseline"] = _guard(lambda: cpu_pfc3d_baseline(args.pfc_n))
            if pfc2d is not None:
                pfc2d["cpu_baseline"] = _guard(cpu_pfc2d_baseline)
            if multi is not None:
                multi["cpu_baseline"] = _guard(cpu_hydro_baseline)
    if ctx.rank == 0:
        print(json.dumps(out))
    if ctx.dist is not None:
        ctx.dist.destroy_process_group()


def main_reference(args):
    """The reference arm: the reference's own CPU implementation of the
    headline step (distfft.forward + inverse over its thread worker group,
    the unmodified package staged at oracle/_ref; the oracle restatement
    when it is absent) on every usable host CPU, same metric / config /
    units as our arm.  Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    n = args.fft_n
    threads = cpu_threads()
    times, kind = ref_fft_roundtrips(n, threads, max(1, args.steps), 150.0)
    s = sum(times) / len(times)
    v = fft_bytes(n) / s / 1e9
    src = ("reference package pfcspectral (oracle/_ref): distfft.forward/inverse over spawn_group"
           if kind == "reference" else "oracle restatement of distfft.py on host threads")
    out = {"impl": "reference", "metric": "distributed 3D FFT GB/s (fp64)", "value": round(v, 4),
           "unit": "GB/s", "n_gpus": world, "steps": len(times), "warmup": args.warmup,
           "ms_per_step": round(s * 1e3, 2), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"3D FFT round trip {n}^3 fp64 (reference C2C slab algorithm on "
                                  f"host threads)", "grid": [n] * 3},
           "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": threads, "kind": kind,
                            "host": cpu_info(),
                            "sample": f"{len(times)} C2C round trips of a real {n}^3 field, {threads} worker "
                                      f"threads ({src}), after one warm-up round trip"},
           "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
