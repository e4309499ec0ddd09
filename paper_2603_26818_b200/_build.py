"""Build libpfcs.so (the sm_100a kernels + C ABI) in-tree with nvcc.

The shared object lands next to this file so it travels with the repo
snapshot to the GPU box.  Objects are compiled in parallel and only rebuilt
when a source or header is newer than the library.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB = PKG / "libpfcs.so"
BUILD = ROOT / "build" / "pfcs"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
              "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; libpfcs cannot be built")
    return cand


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _deps():
    return list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + \
        list(INCLUDE.glob("*.h"))


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in _deps())


def _compile(src: Path, nvcc: str, verbose: bool) -> tuple[Path, str]:
    obj = BUILD / (src.stem + ".o")
    cmd = [nvcc, *ARCH, *NVCC_FLAGS, "-I", str(INCLUDE), "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
    return obj, res.stderr


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    nvcc = _nvcc()
    BUILD.mkdir(parents=True, exist_ok=True)
    srcs = _sources()
    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        futs = [ex.submit(_compile, s, nvcc, verbose) for s in srcs]
        objs = []
        for f in futs:
            obj, log = f.result()
            objs.append(obj)
            logs.append(log)
    (BUILD / "ptxas.log").write_text("\n".join(logs))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-Xcompiler", "-fPIC"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print("\n".join(logs), file=sys.stderr)
    return LIB


def build_variant(name: str, defines: list[str], only: list[str] | None = None,
                  reuse: Path | None = None) -> Path:
    """Experimental build with extra -D flags into libpfcs_<name>.so (for A/B
    timing on the GPU via PFCS_LIB_PATH); not used by the product.  With
    `only` (source stems), the other objects are reused from the main build
    (or from the object directory `reuse`)."""
    nvcc = _nvcc()
    build()
    bdir = ROOT / "build" / name
    bdir.mkdir(parents=True, exist_ok=True)
    flags = [f for f in NVCC_FLAGS if f not in ("-v", "-Xptxas")] + [f"-D{d}" for d in defines]
    procs, objs = [], []
    for src in _sources():
        if only is not None and src.stem not in only:
            objs.append(str((reuse or BUILD) / (src.stem + ".o")))
            continue
        obj = bdir / (src.stem + ".o")
        procs.append(subprocess.Popen([nvcc, *ARCH, *flags, "-I", str(INCLUDE), "-c", str(src), "-o", str(obj)]))
        objs.append(str(obj))
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError(f"variant build {name} failed")
    out = PKG / f"libpfcs_{name}.so"
    subprocess.check_call([nvcc, *ARCH, "-shared", "-o", str(out), *objs])
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
