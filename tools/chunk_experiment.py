"""Experiment: L2-resident chaining of the PFC step's y-fwd -> z-update -> y-inv
passes over chunks of K kx-planes (each plane ny*nz*16 B = 16 MB at 1024^3),
so the z pass reads the y pass's output and the y-inverse reads the z pass's
output while they are still in the 126 MB L2.

    python tools/chunk_experiment.py [n] [K ...]

Prints ms per step for the unchunked 4-kernel step and for each K (CUDA
graph of one step, replayed).  Raw C-ABI calls on synthetic data; not a
bench number.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    ks = [int(k) for k in sys.argv[2:] if not k.startswith('-')] or [1, 2, 4, 8]
    import torch

    from paper_2603_26818_b200 import _native as nat

    torch.cuda.set_device(0)
    nh = n // 2 + 1
    C = torch.complex128
    psi = torch.empty((nh, n, n), dtype=C, device="cuda")
    psi.real.normal_()
    psi.imag.normal_()
    psi.mul_(1e-3)
    buf = torch.empty_like(psi)
    buf.copy_(psi)
    kx = torch.linspace(0, 1, nh, dtype=torch.float64, device="cuda")
    ky = torch.linspace(0, 1, n, dtype=torch.float64, device="cuda")
    diag = torch.zeros(nat.DIAG_SLOTS * 4, dtype=torch.float64, device="cuda")
    plane = n * n

    def st():
        return nat.stream_ptr()

    def yf(p0, k):
        nat.call("pfcs_fft_axis_c2c", nat.ptr(buf) + 16 * p0 * plane, nat.ptr(buf) + 16 * p0 * plane,
                 k, n, n, 1, 1, st())

    def yi(p0, k):
        nat.call("pfcs_fft_axis_c2c", nat.ptr(buf) + 16 * p0 * plane, nat.ptr(buf) + 16 * p0 * plane,
                 k, n, n, 1, 0, st())

    def zu(p0, k):
        off = 16 * p0 * plane
        nat.call("pfcs_pfc_update_z", nat.ptr(buf) + off, nat.ptr(psi) + off, nat.ptr(buf) + off, k, n, n, 1, 1,
                 nat.ptr(kx) + 8 * p0, nat.ptr(ky), nat.ptr(ky), -0.3, 1e-3, nat.ptr(diag), st())

    def cube():
        nat.call("pfcs_pfc_cube_x", nat.ptr(buf), n, n * n, 1, nat.ptr(diag), st())

    def step(k):
        cube()
        if k == 0:
            yf(0, nh)
            zu(0, nh)
            yi(0, nh)
        else:
            for p0 in range(0, nh, k):
                kk = min(k, nh - p0)
                yf(p0, kk)
                zu(p0, kk)
                yi(p0, kk)

    if "--once" in sys.argv:  # for ncu: two plain (ungraphed) steps at the first K
        for _ in range(2):
            step(ks[0])
        torch.cuda.synchronize()
        return
    for k in [0] + ks:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step(k)  # warm (allocations, occupancy caches)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step(k)
        g.replay()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        reps = 5
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        print(f"n={n} K={k if k else 'unchunked'} launches/step={1 + 3 * (1 if k == 0 else -(-nh // k))} "
              f"ms/step={a.elapsed_time(b) / reps:.3f}", flush=True)


if __name__ == "__main__":
    main()
