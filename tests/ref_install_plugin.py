"""pytest plugin (-p ref_install_plugin) for running the reference's OWN unit
tests against this package: before any test module is collected -- they bind
`from annq.codebook import encode_dataset` by name at import -- it imports the
unmodified reference from baseline/_ref and calls install(), so every hot-path
entry point the tests reach is the sm_100a implementation."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def pytest_configure(config):
    for p in (REF, ROOT):
        if p not in sys.path:
            sys.path.insert(0, p)
    import annq  # noqa: F401  (the reference)
    import paper_1509_05194_b200 as da

    patched = da.install()
    config._da_patched = patched
    if not patched:
        raise RuntimeError("install() patched nothing")


def pytest_report_header(config):
    return f"annq hot path patched by paper_1509_05194_b200.install(): {len(config._da_patched)} binding sites"
