"""Host-side logic that needs no GPU: validation, config objects, schedules,
content hashes, file formats, synthetic generators and the drop-in patcher."""

import hashlib
import os
import struct
import sys
import types

import numpy as np
import pytest

import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import synthetic
from paper_1509_05194_b200.validation import check_codes, check_query, check_vectors


class TestSchedule:
    def test_known_answers(self):
        assert da.dimension_schedule(960, 10) == [2, 4, 8, 16, 31, 62, 123, 244, 484, 960]
        assert da.dimension_schedule(128, 10) == [2, 3, 5, 7, 12, 19, 30, 49, 79, 128]
        assert da.dimension_schedule(32, 10) == [2, 3, 4, 6, 8, 12, 17, 23, 32]
        assert da.dimension_schedule(1, 10) == [1]

    @pytest.mark.parametrize("d", [2, 3, 4, 7, 33, 500])
    def test_strictly_increasing_ending_at_d(self, d):
        s = da.dimension_schedule(d)
        assert all(b > a for a, b in zip(s, s[1:])) and s[-1] == d and s[0] >= 1

    def test_rejects_bad(self):
        with pytest.raises(ValueError):
            da.dimension_schedule(0)


class TestValidation:
    def test_vectors(self):
        with pytest.raises(ValueError):
            check_vectors(np.zeros(3))
        with pytest.raises(ValueError):
            check_vectors(np.zeros((0, 3)))
        with pytest.raises(ValueError):
            check_vectors(np.array([[np.nan, 1.0]]))
        assert check_vectors(np.zeros((0, 3)), allow_empty=True).shape == (0, 3)
        assert check_vectors([[1, 2]]).dtype == np.float32

    def test_query_and_codes(self):
        with pytest.raises(ValueError):
            check_query(np.zeros(3), 4)
        with pytest.raises(ValueError):
            check_codes(np.array([[0, 4]]), 4)
        with pytest.raises(ValueError):
            check_codes(np.array([[0, 1]]), 4, m_count=3)

    def test_config(self):
        with pytest.raises(ValueError):
            da.TrainConfig(m_count=0)
        with pytest.raises(ValueError):
            da.TrainConfig(beam_width=0)
        with pytest.raises(ValueError):
            da.TrainConfig(rel_tol=-1)
        assert da.TrainConfig().echo()["beam"] == 10


class TestCodebookObjects:
    def test_shape_checks(self):
        with pytest.raises(ValueError):
            da.Codebook(codewords=np.zeros((2, 3)), order=np.arange(2))
        with pytest.raises(ValueError):
            da.Codebook(codewords=np.zeros((2, 3, 4)), order=np.arange(3))
        b = da.Codebook.zeros(3, 300, 4)
        assert b.code_dtype == np.uint16 and b.codewords.dtype == np.float32

    def test_content_hash_definition(self):
        rng = np.random.default_rng(0)
        cw = rng.standard_normal((3, 5, 7)).astype(np.float32)
        b = da.Codebook(codewords=cw, order=np.array([2, 0, 1]))
        h = hashlib.sha256()
        h.update(struct.pack("<III", 7, 3, 5))
        h.update(cw.astype("<f4").tobytes())
        h.update(np.array([2, 0, 1]).astype("<u4").tobytes())
        assert b.content_hash() == h.digest()

    def test_encoded_dataset(self):
        e = da.EncodedDataset(codes=np.array([[1, 2]], dtype=np.int64), k_count=4)
        assert e.codes.dtype == np.uint8 and e.n == 1 and e.m_count == 2
        with pytest.raises(ValueError):
            da.EncodedDataset(codes=np.array([[1, 2]]), k_count=4, id_map=np.arange(2))

    def test_reorder_by_variance_is_host_bookkeeping(self):
        cw = np.zeros((2, 2, 1), dtype=np.float32)
        cw[0, 1], cw[1, 1] = 1.0, 4.0
        book, perm = da.reorder_by_variance(da.Codebook(codewords=cw, order=np.arange(2)))
        np.testing.assert_array_equal(perm, [1, 0])
        np.testing.assert_array_equal(book.order, [1, 0])


def test_file_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    b = da.Codebook(codewords=rng.standard_normal((3, 5, 7)).astype(np.float32), order=np.array([2, 0, 1]))
    da.write_codebook(tmp_path / "b.hclb", b)
    b2 = da.read_codebook(tmp_path / "b.hclb")
    assert b2.codewords.tobytes() == b.codewords.tobytes() and b2.content_hash() == b.content_hash()
    e = da.EncodedDataset(codes=rng.integers(0, 5, (9, 3)), k_count=5)
    da.write_encoded(tmp_path / "e.hcle", e)
    assert da.read_encoded(tmp_path / "e.hcle").codes.tobytes() == e.codes.tobytes()
    (tmp_path / "bad").write_bytes(b"NOPE" + b"\0" * 16)
    with pytest.raises(da.FormatError) as ei:
        da.read_codebook(tmp_path / "bad")
    assert ei.value.exit_code == 2


class TestSynthetic:
    def test_config_a(self):
        X = synthetic.config_a(n=500)
        assert X.shape == (500, 32) and X.dtype == np.float32
        np.testing.assert_array_equal(X, synthetic.config_a(n=500))

    def test_config_b_integers_in_range(self):
        X = synthetic.config_b(n=3000, chunk=1000)
        assert X.shape == (3000, 128)
        assert X.min() >= 0 and X.max() <= 255 and (X == np.rint(X)).all()
        np.testing.assert_array_equal(X[:1000], synthetic.config_b(n=1000, chunk=1000))

    def test_config_c_range(self):
        X = synthetic.config_c(n=300, chunk=100)
        assert X.shape == (300, 960) and 0.0 <= X.min() and X.max() <= 1.0

    def test_stream_chunks_uint8(self):
        a = synthetic.mixture_b_chunk(3, 0, n=100)
        assert a.dtype == np.uint8 and a.shape == (100, 128)
        np.testing.assert_array_equal(a, synthetic.mixture_b_chunk(3, 0, n=100))
        assert not np.array_equal(a, synthetic.mixture_b_chunk(3, 1, n=100))

    def test_candidates_sorted_distinct(self):
        c = synthetic.config_e_candidates(3, ncand=1000, n_total=10**9)
        assert c.shape == (3, 1000)
        for row in c:
            assert (np.diff(row) > 0).all()


def test_install_patches_every_binding_site(monkeypatch):
    names = {"annq": {}, "annq.codebook": {}, "annq.clustering": {}, "annq.annealing": {},
             "annq.estimators": {}, "annq.cli": {}, "annq.atree": {}, "annq.data": {}}
    for modname in names:
        mod = types.ModuleType(modname)
        for n in da._PATCH_TABLE.get(modname, []):
            setattr(mod, n, object())
        monkeypatch.setitem(sys.modules, modname, mod)
    patched = da.install()
    for modname, attrs in da._PATCH_TABLE.items():
        for a in attrs:
            assert (modname, a) in patched
            assert getattr(sys.modules[modname], a).__module__.startswith("paper_1509_05194_b200")


def _real_reference():
    """The unmodified reference installed untracked under baseline/_ref
    (oracle/ship_reference.sh); None when it is not there."""
    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "annq")):
        return None
    return ref


def test_install_against_the_real_reference(monkeypatch):
    """install() on the real annq: every by-name binding site points at this
    package and the raw-kernel counters are one dict (test_codebook.py:236-243)."""
    ref = _real_reference()
    if ref is None:
        pytest.skip("baseline/_ref not installed (oracle/ship_reference.sh)")
    for k in [k for k in sys.modules if k == "annq" or k.startswith("annq.")]:
        monkeypatch.delitem(sys.modules, k)
    monkeypatch.syspath_prepend(ref)
    import importlib

    annq = importlib.import_module("annq")
    saved = {m: dict(vars(sys.modules[m])) for m in list(sys.modules) if m == "annq" or m.startswith("annq.")}
    from paper_1509_05194_b200 import codebook as ours_cb

    old_counters = ours_cb.DEBUG_COUNTERS
    try:
        patched = da.install()
        assert ("annq.annealing", "improved_kmeans") in patched
        assert ("annq.atree", "adc_table") in patched
        assert annq.encode_dataset is da.encode_dataset
        import annq.codebook as rcb

        assert ours_cb.DEBUG_COUNTERS is rcb.DEBUG_COUNTERS
        rcb.DEBUG_COUNTERS["raw_dim_kernel_calls"] = 0
        ours_cb._raw_kernel(2)
        assert rcb.DEBUG_COUNTERS["raw_dim_kernel_calls"] == 2
    finally:
        ours_cb.DEBUG_COUNTERS = old_counters
        for m, d in saved.items():
            vars(sys.modules[m]).update(d)
