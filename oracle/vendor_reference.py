"""Recipe: stage the reference package and its test suite under oracle/_ref/.

TEST INFRASTRUCTURE ONLY (the checker, never the product).  The reference
(`pfcspectral`, pure Python + numpy) is read-only at /root/reference and does
not exist on the GPU box, so this recipe copies — into the git-ignored
oracle/_ref/, which travels with the gpurun snapshot like a built .so —

  oracle/_ref/pfcspectral/   the unmodified reference package
                             (/root/reference/pkg/src/pfcspectral), timed by
                             `bench.py --impl reference` and by bench.py's
                             cpu_baseline legs through its own public API;
  oracle/_ref/refsuite/      the reference's own test suite
                             (/root/reference/pkg/tests) plus
                             oracle/refsuite_conftest.py as its conftest.py,
                             which aliases `pfcspectral` to this repo's
                             package so the suite exercises the B200 path
                             (tests/test_gpu_reference_suite.py runs it).

Nothing is committed from /root/reference: oracle/_ref/ is in .gitignore.
Run by __graft_entry__.build() when /root/reference is present; idempotent.
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg")
OUT = HERE / "_ref"


def stage(ref: Path = REF, out: Path = OUT) -> bool:
    src_pkg = ref / "src" / "pfcspectral"
    src_tests = ref / "tests"
    if not src_pkg.is_dir() or not src_tests.is_dir():
        return False
    out.mkdir(parents=True, exist_ok=True)
    dst_pkg = out / "pfcspectral"
    if dst_pkg.exists():
        shutil.rmtree(dst_pkg)
    shutil.copytree(src_pkg, dst_pkg, ignore=shutil.ignore_patterns("__pycache__"))
    suite = out / "refsuite"
    if suite.exists():
        shutil.rmtree(suite)
    shutil.copytree(src_tests, suite, ignore=shutil.ignore_patterns("__pycache__"))
    shutil.copy(HERE / "refsuite_conftest.py", suite / "conftest.py")
    for p in [dst_pkg, suite, *dst_pkg.rglob("*"), *suite.rglob("*")]:  # copies of a read-only tree
        p.chmod(0o755 if p.is_dir() else 0o644)
    (out / "SOURCE.txt").write_text(f"copied from {ref} by oracle/vendor_reference.py\n")
    return True


if __name__ == "__main__":
    ok = stage()
    print("staged" if ok else "reference not present", OUT)
    sys.exit(0 if ok else 1)
