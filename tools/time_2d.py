"""Time configs[0] (2D PFC 256^2, R2C, 100-step pfc_run blocks) on cuda:0:
    python tools/time_2d.py [reps]      (environment switches apply: PFCS_TMA, PFCS_PDL, ...)"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import paper_2603_26818_b200 as pkg
    from paper_2603_26818_b200 import distfft, pfc

    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    n = (256, 256, 1)
    grid = pkg.GridSpec(n, pfc.default_domain_length(n))
    psi0 = pfc.initial_field("constant_plus_noise", grid, seed=0, noise_amplitude=0.01)

    def body(w):
        f = distfft.scatter(psi0, w, grid, distfft.Layout.Y_SLAB, real=True)
        st = pfc.PfcState(psi_hat=distfft.forward(f, w), grid=grid, symbols=pkg.make_symbols(grid, -0.3), worker=w)
        pfc.pfc_run(st, pfc.PfcParams(), 100)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        out = []
        for _ in range(reps):
            a.record()
            pfc.pfc_run(st, pfc.PfcParams(), 100)
            b.record()
            torch.cuda.synchronize()
            out.append(a.elapsed_time(b) * 10.0)  # us per step
        return min(out)

    us = pkg.spawn_group(1, body)[0]
    print(f"2D 256^2: {us:.2f} us/step", {k: v for k, v in os.environ.items() if k.startswith("PFCS_")})


if __name__ == "__main__":
    main()
