"""Run the 1024^3 PFC step loop for ~`secs` seconds while sampling power,
clocks and throttle reasons with nvidia-smi (diagnostic, not a bench)."""
import subprocess
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
    import torch

    from paper_2603_26818_b200 import distfft, pfc
    from paper_2603_26818_b200.grid import GridSpec, make_symbols
    from paper_2603_26818_b200.transport import Worker, WorkerGroup

    n = 1024
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    w = Worker(WorkerGroup(1), 0, dev)
    grid = GridSpec((n,) * 3, pfc.default_domain_length((n,) * 3))
    psi0 = (-0.31 + 0.02 * torch.rand((n,) * 3, dtype=torch.float64, device=dev)).contiguous()
    spec = distfft.forward(distfft.DistField(grid, distfft.Layout.Z_SLAB, distfft.Space.PHYSICAL, psi0), w)
    del psi0
    sym = make_symbols(grid, -0.3, layout=distfft._layout(grid, distfft.Layout.X_SLAB, 1, True), rank=0)
    st = pfc.PfcState(psi_hat=spec, grid=grid, symbols=sym, worker=w)
    pfc.pfc_run(st, pfc.PfcParams(), 3)
    torch.cuda.synchronize()
    samples = []
    stop = threading.Event()

    def sampler():
        q = "power.draw,power.limit,clocks.sm,clocks.mem,clocks_throttle_reasons.active,temperature.gpu"
        while not stop.is_set():
            out = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-i", "0"],
                                 capture_output=True, text=True).stdout.strip()
            samples.append(out)
            time.sleep(0.1)

    th = threading.Thread(target=sampler, daemon=True)
    th.start()
    t0 = time.time()
    steps = 0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    while time.time() - t0 < secs:
        pfc.pfc_run(st, pfc.PfcParams(), 20)
        steps += 20
    b.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    print(f"{steps} steps, {a.elapsed_time(b) / steps:.3f} ms/step")
    for s in samples[:: max(1, len(samples) // 12)]:
        print(s)


if __name__ == "__main__":
    main()
