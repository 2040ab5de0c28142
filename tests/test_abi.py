"""The C-ABI library: builds for sm_100a, loads without a GPU, exports every
symbol include/da_b200.h declares, and the Python layer binds all of them."""

import os
import re
import subprocess

import numpy as np
import pytest
import torch

from paper_1509_05194_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "da_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(da_\w+)\s*\(", text, flags=re.M)))


def test_header_lists_the_hot_path():
    names = declared()
    for must in ("da_assign", "da_group_sums", "da_heat_up", "da_pca_cov", "da_rotate", "da_cross_products",
                 "da_encode", "da_pair_sums", "da_adc_lut", "da_adc_scan", "da_adc_pack", "da_unpack_vecs", "da_assign_bind_image", "da_assign_image_bytes",
                 "da_adc_scan_packed", "da_atree_search", "da_knn", "da_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (da_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    for n in declared():
        getattr(lib, n)


def test_python_binds_every_declared_symbol():
    assert set(declared()) == set(_native.EXPORTED)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_plumbing_without_gpu():
    lib = _native.load_library()
    assert lib.da_version() == 1
    assert _native.launch_count() >= 0
    # argument validation happens before any device work -> ValueError, message kept
    with pytest.raises(ValueError, match="beam_width"):
        _native.native.da_encode(None, 1, 1, 1, 1, None, 1, 1, 0, None, None, None, 1, 1, None, None)
    assert b"beam_width" in lib.da_last_error()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    import paper_1509_05194_b200 as da

    book = da.Codebook.zeros(2, 4, 3)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        da.encode_dataset(book, np.zeros((5, 3), dtype=np.float32))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        da.train_from_scratch(np.zeros((10, 3), dtype=np.float32), da.TrainConfig(m_count=1, k_count=2))
