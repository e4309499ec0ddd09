"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python oracle/gen_golden.py

It imports `pfcspectral` from /root/reference/pkg/src (read-only, not copied)
and writes small .npz fixtures to tests/golden/.  These pin both the numpy
oracle (oracle/ref_numpy.py) and the CUDA path; nothing on the GPU box reads
/root/reference.
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main() -> None:
    sys.path.insert(0, str(REF))
    import pfcspectral as ref  # noqa: E402
    from pfcspectral import distfft, pfc, hydro  # noqa: E402
    from pfcspectral.grid import GridSpec, make_symbols  # noqa: E402

    OUT.mkdir(parents=True, exist_ok=True)

    # 1. serial transforms incl. non-power-of-two and prime lengths
    rng = np.random.default_rng(2026)
    fx = {}
    for i, shape in enumerate([(5, 6, 7), (8, 8, 8), (16, 4, 3), (12, 1, 1), (3, 32, 2), (64, 2, 16)]):
        a = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        fx[f"in{i}"] = a
        fx[f"nd{i}"] = ref.fft_nd(a)
        fx[f"ind{i}"] = ref.fft_nd(a, forward=False)
        for ax in range(3):
            fx[f"ax{i}_{ax}"] = ref.fft_axis(a, ax)
    np.savez_compressed(OUT / "fft_serial.npz", **fx)

    # 2. distributed forward on uneven splits (G = 3) vs the reference
    dx = {}
    for i, shape in enumerate([(8, 12, 16), (10, 10, 10), (6, 9, 1)]):
        grid = GridSpec(shape, (1.0, 1.0, 1.0))
        a = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)

        def body(w, a=a, grid=grid):
            f = distfft.scatter(a, w, grid, distfft.physical_layout(grid))
            return distfft.gather(distfft.forward(f, w), w)

        dx[f"in{i}"] = a
        dx[f"out{i}"] = ref.spawn_group(3, body)[0]
    np.savez_compressed(OUT / "fft_dist.npz", **dx)

    # 3. PFC runs: configs[0] (2D 256^2, 100 steps) and a 3D 32^3 run
    def pfc_run(n, steps, workers, seed=0, kind="constant_plus_noise", **kw):
        grid = GridSpec(n, pfc.default_domain_length(n))
        params = pfc.PfcParams(eps=-0.3, dt=0.1, psi_bar=-0.3, n_steps=steps)

        def body(w):
            xlay = distfft.layout_for(grid, distfft.Layout.X_SLAB, w.size)
            sym = make_symbols(grid, params.eps, layout=xlay, rank=w.rank)
            f0 = pfc.init_condition(kind, grid, w, psi_bar=params.psi_bar, seed=seed, **kw)
            st = pfc.PfcState(psi_hat=distfft.forward(f0, w), grid=grid, symbols=sym, worker=w)
            energies = [pfc.free_energy(st, params)]
            means = [pfc.mean_and_max(st)]
            for s in range(steps):
                pfc.pfc_step(st, params)
                if (s + 1) % 20 == 0:
                    energies.append(pfc.free_energy(st, params))
                    means.append(pfc.mean_and_max(st))
            psi = distfft.gather(distfft.inverse(st.psi_hat, w), w)
            return psi, energies, means

        psi, e, m = ref.spawn_group(workers, body)[0]
        init = pfc.initial_field(kind, grid, psi_bar=-0.3, seed=seed, **kw)
        return dict(init=init, psi=psi.real, energies=np.array(e), means=np.array(m),
                    length=np.array(grid.length))

    np.savez_compressed(OUT / "pfc2d_256.npz", **pfc_run((256, 256, 1), 100, 1, noise_amplitude=0.01))
    np.savez_compressed(OUT / "pfc3d_32.npz", **pfc_run((32, 32, 32), 100, 2, noise_amplitude=0.01))
    np.savez_compressed(OUT / "pfc3d_fcc16.npz",
                        **pfc_run((16, 16, 16), 40, 1, kind="two_mode_fcc_3d", amplitude=0.05))

    # 4. hydro serial dataflow (hydro.py:110-126) on 16^3 FCC
    n = (16, 16, 16)
    grid = GridSpec(n, (2 * math.pi * math.sqrt(3),) * 3)
    hp = hydro.HydroParams(pfc=pfc.PfcParams(eps=-0.3, dt=0.1, psi_bar=-0.3, n_steps=10),
                           rho=1.0, gamma=1.0, a0=2.0)
    sym = make_symbols(grid, -0.3, a0=2.0)
    psi0 = pfc.initial_field("two_mode_fcc_3d", grid, psi_bar=-0.3, amplitude=0.05, seed=2)
    psi_hat = ref.fft_nd(psi0.astype(np.complex128))
    zeros = np.zeros(n, dtype=np.complex128)
    fields = hydro.HydroFields(psi_hat=psi_hat, psi=ref.fft_nd(psi_hat, forward=False),
                               v_hat=[zeros.copy() for _ in range(3)], v=[zeros.copy() for _ in range(3)])
    for _ in range(10):
        hydro.serial_hydro_step(fields, sym, hp)
    np.savez_compressed(OUT / "hydro16.npz", psi0=psi0, psi_hat=fields.psi_hat, psi=fields.psi,
                        v1=fields.v[0], v2=fields.v[1], v3=fields.v[2],
                        vh1=fields.v_hat[0], vh2=fields.v_hat[1], vh3=fields.v_hat[2])

    # 5. initial conditions (setup generators pinned bit-for-bit)
    g3 = GridSpec((8, 8, 8), (2 * math.pi * math.sqrt(3),) * 3)
    g2 = GridSpec((32, 32, 1), pfc.default_domain_length((32, 32, 1)))
    np.savez_compressed(
        OUT / "init.npz",
        noise=pfc.initial_field("constant_plus_noise", g3, seed=42),
        crystallites=pfc.initial_field("seeded_crystallites", g3, seed=42, n_seeds=3),
        fcc=pfc.initial_field("two_mode_fcc_3d", g3, amplitude=0.07),
        tri=pfc.initial_field("single_mode_triangular_2d", g2, amplitude=0.3, psi_bar=-0.2),
        tri_seeds=pfc.initial_field("seeded_crystallites", g2, seed=7, n_seeds=2),
    )
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
