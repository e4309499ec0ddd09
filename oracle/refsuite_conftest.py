"""conftest.py for the reference's own test suite staged at
oracle/_ref/refsuite/ (oracle/vendor_reference.py).  TEST INFRASTRUCTURE.

Aliases the reference package name `pfcspectral` (and every submodule the
suite imports) to this repo's drop-in package, so the reference tests run
unmodified against the B200 path (SURVEY.md App. C API).  The CLI module is
out of scope (control plane): test_cli.py is ignored by the runner.
"""

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[3]  # oracle/_ref/refsuite -> repo root
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

_pkg = importlib.import_module("paper_2603_26818_b200")
sys.modules["pfcspectral"] = _pkg
for _m in ("grid", "fftcore", "transport", "distfft", "pfc", "hydro", "config", "snapshot", "run", "bench"):
    sys.modules[f"pfcspectral.{_m}"] = importlib.import_module(f"paper_2603_26818_b200.{_m}")
