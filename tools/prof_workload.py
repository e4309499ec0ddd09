"""Run the bench workloads once, for `ncu` captures of exactly one step.

    python tools/prof_workload.py fft [n]    # 1 warm + 1 measured 3D R2C/C2R round trip
    python tools/prof_workload.py pfc [n]    # setup forward + 1 warm + 1 measured PFC step
    python tools/prof_workload.py multi [n]  # 2 serial multiphysics steps (5 fields, 512^3 default)

Kernel launch order (for ncu --launch-skip / --launch-count):
  fft: warm round trip = 6 launches (rfft_x, y fwd, z fwd, z inv, y inv, irfft_x),
       then the measured 6.
  pfc: setup forward = 3 launches (rfft_x, y fwd, z fwd), warm step = 4
       (pfc_update_z, y inv, cube_x, y fwd), then the measured 4.
Same package API and inputs as bench.py (synthetic, seeded on device).
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    what = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else (1024 if what == "pfc" else 512)
    import torch

    from paper_2603_26818_b200 import distfft, pfc
    from paper_2603_26818_b200.grid import GridSpec, make_symbols
    from paper_2603_26818_b200.transport import Worker, WorkerGroup

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    w = Worker(WorkerGroup(1), 0, dev)
    if True:
        if what == "fft":
            grid = GridSpec((n, n, n), (1.0, 1.0, 1.0))
            gen = torch.Generator(device=dev).manual_seed(1234)
            x = torch.randn((n, n, n), dtype=torch.float64, device=dev, generator=gen)
            f = distfft.DistField(grid, distfft.Layout.Z_SLAB, distfft.Space.PHYSICAL, x)
            for _ in range(2):
                s = distfft.forward(f, w)
                f = distfft.inverse(s, w)
        elif what == "multi":
            import numpy as np

            from paper_2603_26818_b200 import hydro, multiphysics as mpx

            grid = GridSpec((n,) * 3, (2 * np.pi * np.sqrt(3) * (n // 8),) * 3)
            hp = hydro.HydroParams(pfc=pfc.PfcParams(eps=-0.3, dt=0.1), rho=1.0, gamma=1.0, a0=2.0)
            mp = mpx.MultiParams(hydro=hp, mobility=1.0, kappa=1.0, alpha=1.0, beta=0.0)
            sym = make_symbols(grid, -0.3, a0=2.0)
            gen = torch.Generator(device=dev).manual_seed(11)
            C = torch.complex128

            def field(scale, base=0.0):
                x = torch.rand((n,) * 3, dtype=torch.float64, device=dev, generator=gen)
                return (base + scale * (x - 0.5)).to(C)

            psi, c = field(0.02, -0.3), field(0.2)
            zeros = torch.zeros((n,) * 3, dtype=C, device=dev)
            f = mpx.MultiFields(psi_hat=hydro._fft(psi, True), psi=psi, c_hat=hydro._fft(c, True), c=c,
                                v_hat=[zeros.clone() for _ in range(3)], v=[zeros.clone() for _ in range(3)])
            for _ in range(2):
                mpx.serial_multi_step(f, sym, mp)
        else:
            grid = GridSpec((n, n, n), pfc.default_domain_length((n, n, n)))
            gen = torch.Generator(device=dev).manual_seed(7)
            psi0 = torch.rand((n, n, n), dtype=torch.float64, device=dev, generator=gen)
            psi0.mul_(0.02).add_(-0.31)
            f0 = distfft.DistField(grid, distfft.Layout.Z_SLAB, distfft.Space.PHYSICAL, psi0)
            spec = distfft.forward(f0, w)
            del f0, psi0
            hl = distfft._layout(grid, distfft.Layout.X_SLAB, 1, True)
            sym = make_symbols(grid, -0.3, layout=hl, rank=0)
            st = pfc.PfcState(psi_hat=spec, grid=grid, symbols=sym, worker=w)
            pfc.pfc_run(st, pfc.PfcParams(), 2)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
