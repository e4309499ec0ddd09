import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpfcs.so")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(GOLDEN / f"{name}.npz"))
        return cache[name]

    return load


def rel_inf(a, b):
    import numpy as np

    scale = float(np.max(np.abs(b))) if np.size(b) else 0.0
    err = float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) if np.size(b) else 0.0
    return err / scale if scale else err


def rel_l2(a, b):
    import numpy as np

    nb = float(np.linalg.norm(np.ravel(b)))
    d = float(np.linalg.norm(np.ravel(np.asarray(a) - np.asarray(b))))
    return d / nb if nb else d
