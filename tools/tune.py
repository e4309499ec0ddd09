"""Tile-width / pipeline-depth sweep for the libpfcs pass kernels (run on a B200).

Builds (or reuses) paper_2603_26818_b200/libpfcs_tune.so compiled with
-DPFCS_TUNE, then times each kernel kind at the bench sizes for variants 0..7
(T = T_MIN << (v & 3), 1 + (v >> 2) cp.async stages) with CUDA events and prints a JSON table.  The best
variants are baked into default_variant() (csrc/pfcs_internal.h).
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
TUNE_LIB = ROOT / "paper_2603_26818_b200" / "libpfcs_tune.so"


def build_tune():
    from paper_2603_26818_b200 import _build
    objs = []
    bdir = ROOT / "build" / "tune"
    bdir.mkdir(parents=True, exist_ok=True)
    nvcc = _build._nvcc()
    procs = []
    for src in _build._sources():
        obj = bdir / (src.stem + ".o")
        cmd = [nvcc, *_build.ARCH, *[f for f in _build.NVCC_FLAGS if f not in ("-v", "-Xptxas")], "-DPFCS_TUNE",
               "-I", str(_build.INCLUDE), "-c", str(src), "-o", str(obj)]
        procs.append(subprocess.Popen(cmd))
        objs.append(str(obj))
    for p in procs:
        assert p.wait() == 0
    subprocess.check_call([nvcc, *_build.ARCH, "-shared", "-o", str(TUNE_LIB), *objs])


def main():
    if "--build" in sys.argv:
        build_tune()
        return
    os.environ.setdefault("PFCS_LIB_PATH", str(TUNE_LIB))
    kinds = None
    sizes = (512, 1024)
    for a in sys.argv[1:]:
        if a.startswith("--kinds="):
            kinds = {int(k) for k in a.split("=", 1)[1].split(",")}
        if a.startswith("--sizes="):
            sizes = tuple(int(k) for k in a.split("=", 1)[1].split(","))
    import torch
    from paper_2603_26818_b200 import _native as nat

    torch.cuda.set_device(0)
    st = nat.stream_ptr()

    def time_it(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    results = {}
    C = torch.complex128

    def sweep(kind, n, fn, nbytes):
        if kinds is not None and kind not in kinds:
            return
        row = {}
        for s in range(8):
            os.environ[f"PFCS_VARIANT_{kind}_{n}"] = str(s)
            try:
                ms = time_it(fn)
                row[s] = round(nbytes / (ms * 1e-3) / 1e9, 1)
            except Exception as e:  # tile too large etc.
                row[s] = None
                print("  variant", s, "failed:", str(e)[:120], flush=True)
        del os.environ[f"PFCS_VARIANT_{kind}_{n}"]
        results[f"{kind}_{n}"] = row
        print(kind, n, row, flush=True)

    for n in sizes:
        nh = n // 2 + 1
        # LINES (z pass, plain)
        a = torch.empty(nh * n * n, dtype=C, device="cuda")
        a.real.normal_()
        sweep(0, n, lambda: nat.call("pfcs_fft_zlines", nat.ptr(a), nat.ptr(a), nh * n, n, 1, 1, 1, st),
              2 * 16 * a.numel())
        # STRIDED (y pass)
        sweep(1, n, lambda: nat.call("pfcs_fft_axis_c2c", nat.ptr(a), nat.ptr(a), nh, n, n, 1, 1, st),
              2 * 16 * a.numel())
        # REALX (R2C along x), M = n/2
        r = torch.randn(n * n * n, dtype=torch.float64, device="cuda")
        sweep(2, n // 2, lambda: nat.call("pfcs_rfft_x", nat.ptr(r), nat.ptr(a), n, n * n, st),
              8 * r.numel() + 16 * a.numel())
        # C2R along x shares the REALX variant key; reported as kind 6
        if kinds is None or 6 in kinds:
            kinds_save = kinds
            kinds = None
            row_key = f"2_{n // 2}"
            prev = results.pop(row_key, None)
            sweep(2, n // 2, lambda: nat.call("pfcs_irfft_x", nat.ptr(a), nat.ptr(r), n, n * n, st),
                  8 * r.numel() + 16 * a.numel())
            results[f"6_{n // 2}"] = results.pop(row_key)
            if prev is not None:
                results[row_key] = prev
            kinds = kinds_save
        del r
        diag = torch.zeros(nat.DIAG_SLOTS * 4, dtype=torch.float64, device="cuda")
        # fused cube pass (KIND_CUBER = 5, keyed by M)
        sweep(5, n // 2, lambda: nat.call("pfcs_pfc_cube_x", nat.ptr(a), n, n * n, 1, nat.ptr(diag), st),
              2 * 16 * a.numel())
        # PFCZ (fused update)
        psi = torch.empty_like(a)
        psi.real.normal_()
        kx = torch.linspace(0, 1, nh, dtype=torch.float64, device="cuda")
        ky = torch.linspace(0, 1, n, dtype=torch.float64, device="cuda")
        sweep(4, n, lambda: nat.call("pfcs_pfc_update_z", nat.ptr(a), nat.ptr(psi), nat.ptr(a), nh, n, n, 1, 1,
                                     nat.ptr(kx), nat.ptr(ky), nat.ptr(ky), -0.3, 1e-9, nat.ptr(diag), st),
              4 * 16 * a.numel())
        del a, psi
        torch.cuda.empty_cache()
    print(json.dumps({"lib": os.environ["PFCS_LIB_PATH"].rsplit("/", 1)[-1], "results": results}))


if __name__ == "__main__":
    main()
