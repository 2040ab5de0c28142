import os
import sys

# The golden fixtures were produced by the reference with numpy's bundled
# OpenBLAS running its SkylakeX kernels (oracle/make_golden.py records this in
# tests/golden/meta.json).  LAPACK's eigh, which both the reference and this
# build run on the host, depends on those kernels at the ulp level, so the
# test process pins the same core type before numpy loads.
os.environ.setdefault("OPENBLAS_CORETYPE", "SkylakeX")

import numpy as np  # noqa: E402
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libda_b200.so")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.fail(f"golden fixture {name} missing (python oracle/make_golden.py)")
    return np.load(path)


@pytest.fixture(scope="session")
def golden():
    return load_golden
