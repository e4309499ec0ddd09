"""Time the 512^3 serial R2C multiphysics step (bench.py's configs[4] line)
on cuda:0:   python tools/time_multi.py [n] [steps]   (env switches apply)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import numpy as np
    import torch

    from paper_2603_26818_b200 import hydro, multiphysics as mpx
    from paper_2603_26818_b200.grid import GridSpec, make_symbols
    from paper_2603_26818_b200.pfc import PfcParams

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    grid = GridSpec((n,) * 3, (2 * np.pi * np.sqrt(3) * (n // 8),) * 3)
    hp = hydro.HydroParams(pfc=PfcParams(eps=-0.3, dt=0.1), rho=1.0, gamma=1.0, a0=2.0)
    mp = mpx.MultiParams(hydro=hp, mobility=1.0, kappa=1.0, alpha=1.0, beta=0.0)
    sym = make_symbols(grid, -0.3, a0=2.0)
    g = torch.Generator(device=dev).manual_seed(11)
    psi = -0.3 + 0.02 * (torch.rand((n,) * 3, dtype=torch.float64, device=dev, generator=g) - 0.5)
    c = 0.2 * (torch.rand((n,) * 3, dtype=torch.float64, device=dev, generator=g) - 0.5)
    R = mpx._Real3.of((n,) * 3, sym, dev)
    z = torch.zeros_like(psi)
    f = mpx.MultiFields(psi_hat=R.fwd(psi), psi=psi, c_hat=R.fwd(c), c=c, v_hat=[R.fwd(z) for _ in range(3)],
                        v=[z.clone() for _ in range(3)])
    for _ in range(2):
        mpx.serial_multi_step(f, sym, mp)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        mpx.serial_multi_step(f, sym, mp)
    b.record()
    torch.cuda.synchronize()
    print(f"multiphysics {n}^3: {a.elapsed_time(b) / steps:.3f} ms/step",
          {k: v for k, v in os.environ.items() if k.startswith("PFCS_")})


if __name__ == "__main__":
    main()
