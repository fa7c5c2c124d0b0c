import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


def load_golden():
    """Golden cases produced by the reference itself (tests/golden/make_golden.py)."""
    z = np.load(GOLDEN)
    cases = {}
    for k in z.files:
        p, name = k[:3], k[4:]
        cases.setdefault(p, {})[name] = z[k]
    out = []
    for p in sorted(cases):
        c = cases[p]
        c["kind"] = str(c["kind"])
        c["dims"] = tuple(int(d) for d in c["dims"])
        c["h"] = float(c["h"])
        out.append(c)
    return out


@pytest.fixture(scope="session")
def golden():
    return load_golden()
