"""The reference's own unit tests (pkg/tests of annq), run unmodified with the
hot path patched to this package by install().  The reference is
shipped untracked under baseline/_ref by oracle/ship_reference.sh; a box
without it skips.  Each file runs in its own subprocess so the patched
reference never leaks into this process."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "annq_tests")

# the hot-path suites of SURVEY 8(b)/(c); test_acceptance criteria 1-3 are the
# beam/oracle equivalence, ADC exactness and DA monotonicity checks
SUITES = [
    ("test_codebook.py", None),
    ("test_clustering.py", None),
    ("test_annealing.py", None),
    ("test_acceptance.py", "criterion_1 or criterion_2 or criterion_3"),
]


@pytest.mark.parametrize("fname,select", SUITES, ids=[s[0] for s in SUITES])
def test_reference_suite_under_install(fname, select):
    path = os.path.join(REF_TESTS, fname)
    if not os.path.exists(path):
        pytest.skip("baseline/_ref not shipped (oracle/ship_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), ROOT, os.path.join(ROOT, "baseline", "_ref")]
                                        + ([env["PYTHONPATH"]] if env.get("PYTHONPATH") else []))
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", path, "-q", "-p", "ref_install_plugin", "-p", "no:cacheprovider",
           "--rootdir", REF_TESTS, "-x"]
    if select:
        cmd += ["-k", select]
    r = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=1800)
    tail = (r.stdout[-4000:] + "\n" + r.stderr[-2000:])
    assert r.returncode == 0, tail
    assert "passed" in r.stdout, tail
