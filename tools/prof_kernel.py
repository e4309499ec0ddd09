"""Launch one libpfcs pass kernel at a bench size, for `ncu --set full` captures.

    python tools/prof_kernel.py <kind> [n] [reps]

kind: cube_x | update_z | rfft_x | irfft_x | rfft_pro{0,1,3} | deriv<axis><aux_axis> | zlines | strided
The kernel runs `reps` times (default 2: one warm launch + one to capture with
`ncu -k regex:<kernel> -s 1 -c 1`).  Prints the average CUDA-event time of
launches 2..reps (never a bench number when run under ncu).
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    kind = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    import torch
    from paper_2603_26818_b200 import _native as nat

    torch.cuda.set_device(0)
    st = nat.stream_ptr()
    nh = n // 2 + 1
    C = torch.complex128
    a = torch.empty(nh * n * n, dtype=C, device="cuda")
    a.real.normal_()
    a.imag.normal_()
    diag = torch.zeros(nat.DIAG_SLOTS * 4, dtype=torch.float64, device="cuda")
    if kind == "cube_x":
        fn = lambda: nat.call("pfcs_pfc_cube_x", nat.ptr(a), n, n * n, 1, nat.ptr(diag), st)
    elif kind == "update_z":
        psi = torch.empty_like(a)
        psi.real.normal_()
        kx = torch.linspace(0, 1, nh, dtype=torch.float64, device="cuda")
        ky = torch.linspace(0, 1, n, dtype=torch.float64, device="cuda")
        fn = lambda: nat.call("pfcs_pfc_update_z", nat.ptr(a), nat.ptr(psi), nat.ptr(a), nh, n, n, 1, 1,
                              nat.ptr(kx), nat.ptr(ky), nat.ptr(ky), -0.3, 1e-9, nat.ptr(diag), st)
    elif kind in ("rfft_x", "irfft_x"):
        r = torch.randn(n * n * n, dtype=torch.float64, device="cuda")
        if kind == "rfft_x":
            fn = lambda: nat.call("pfcs_rfft_x", nat.ptr(r), nat.ptr(a), n, n * n, st)
        else:
            fn = lambda: nat.call("pfcs_irfft_x", nat.ptr(a), nat.ptr(r), n, n * n, st)
    elif kind.startswith("rfft_pro"):  # rfft_pro0 / rfft_pro1 / rfft_pro3: R2C x pass with a prologue
        r = torch.randn(n * n * n, dtype=torch.float64, device="cuda")
        aux = torch.randn_like(r)
        pk = int(kind[-1])
        fn = lambda: nat.call("pfcs_rfft_x_pro", nat.ptr(r), nat.ptr(a), n, n * n, pk, nat.ptr(aux), 0.5, st)
    elif kind.startswith("deriv"):  # deriv<axis><aux_axis>: an inverse pass with the i d multiplier fused
        ax, aa = int(kind[5]), int(kind[6])
        d = torch.randn(n if aa else nh, dtype=torch.float64, device="cuda")
        b = torch.empty_like(a)
        fn = lambda: nat.call("pfcs_fft_axis_c2c_pro", nat.ptr(a), nat.ptr(b), nh, n, n, ax, 0, 3, nat.ptr(d), aa, st)
    elif kind == "zlines":
        fn = lambda: nat.call("pfcs_fft_zlines", nat.ptr(a), nat.ptr(a), nh * n, n, 1, 1, 1, st)
    elif kind == "xdot3":  # fused advection x pass over three stacked derivative spectra
        s3 = torch.empty(3 * nh * n * n, dtype=C, device="cuda")
        s3.real.normal_()
        s3.imag.normal_()
        vv = [torch.randn(n * n * n, dtype=torch.float64, device="cuda") for _ in range(3)]
        s3v = s3.view(3, -1)
        fn = lambda: nat.call("pfcs_xdot3_x", nat.ptr(s3v[0]), nat.ptr(s3v[1]), nat.ptr(s3v[2]), nat.ptr(vv[0]),
                              nat.ptr(vv[1]), nat.ptr(vv[2]), nat.ptr(a), n, n * n, None, st)
    elif kind == "xmul":
        g = torch.randn(n * n * n, dtype=torch.float64, device="cuda")
        fn = lambda: nat.call("pfcs_xmul_x", nat.ptr(a), nat.ptr(g), n, n * n, st)
    elif kind == "mu_z":  # mu_hat with its operands' forward z passes
        f2 = a.clone()
        mu = torch.empty_like(a)
        kxv = torch.linspace(0, 1, nh, dtype=torch.float64, device="cuda")
        kyv = torch.linspace(0, 1, n, dtype=torch.float64, device="cuda")
        fn = lambda: nat.call("pfcs_hydro_mu_z", nat.ptr(a), nat.ptr(f2), nat.ptr(mu), None, nh, n, n, nat.ptr(kxv),
                              nat.ptr(kyv), nat.ptr(kyv), -0.3, st)
    elif kind == "strided_oop":
        b = torch.empty_like(a)
        fn = lambda: nat.call("pfcs_fft_axis_c2c", nat.ptr(a), nat.ptr(b), nh, n, n, 1, 0, st)
    elif kind == "strided":
        fn = lambda: nat.call("pfcs_fft_axis_c2c", nat.ptr(a), nat.ptr(a), nh, n, n, 1, 1, st)
    else:
        raise SystemExit(f"unknown kind {kind}")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    fn()
    ev[0].record()
    for i in range(reps - 1):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / max(reps - 1, 1)
    print(kind, n, "avg launch ms", round(ms, 4), "env",
          {k: v for k, v in os.environ.items() if k.startswith("PFCS_")})


if __name__ == "__main__":
    main()
