"""Host readers/writers of texmex record files and HCLE streaming (SURVEY §8f
row 4), mirroring the reference's own data tests (pkg/tests/test_data.py) plus
the streaming pieces: chunked header checks and the chunked HCLE writer."""

import struct

import numpy as np
import pytest

from paper_1509_05194_b200 import Codebook, EncodedDataset, FormatError, read_encoded, write_encoded
from paper_1509_05194_b200.codebook import EncodedWriter
from paper_1509_05194_b200.data import VecsFile, read_bvecs, read_fvecs, read_ivecs, write_fvecs, write_ivecs


def test_fvecs_single_record_and_empty(tmp_path):
    p = tmp_path / "one.fvecs"
    p.write_bytes(struct.pack("<i2f", 2, 1.0, 2.0))
    X = read_fvecs(p)
    assert X.dtype == np.float32 and X.shape == (1, 2)
    np.testing.assert_array_equal(X, [[1.0, 2.0]])
    e = tmp_path / "empty.fvecs"
    e.write_bytes(b"")
    assert read_fvecs(e).shape == (0, 0)


@pytest.mark.parametrize("payload,msg", [
    (struct.pack("<if", 2, 1.0) + b"\x01", "truncated record at byte offset 4"),
    (struct.pack("<i2f", 2, 1.0, 2.0) + struct.pack("<i3f", 3, 1.0, 2.0, 3.0),
     "inconsistent dimensions 2 and 3 at byte offset 12"),
    (struct.pack("<i", 0), "invalid dimension header 0 at byte offset 0"),
    (b"\x01\x00", "truncated record header at byte offset 0"),
    (struct.pack("<i2f", 2, 1.0, 2.0) + b"\x02\x00", "truncated record header at byte offset 12"),
])
def test_fvecs_format_errors(tmp_path, payload, msg):
    p = tmp_path / "bad.fvecs"
    p.write_bytes(payload)
    with pytest.raises(FormatError, match=msg):
        read_fvecs(p)


def test_fvecs_nonfinite_and_round_trip(tmp_path):
    p = tmp_path / "nan.fvecs"
    p.write_bytes(struct.pack("<i2f", 2, 1.0, float("nan")))
    with pytest.raises(FormatError, match="non-finite value in payload"):
        read_fvecs(p)
    rng = np.random.default_rng(0)
    for n, d in [(17, 5), (1, 1), (8, 6)]:
        X = (rng.standard_normal((n, d)) * 100).astype(np.float32)
        q = tmp_path / f"rt{n}.fvecs"
        write_fvecs(q, X)
        assert read_fvecs(q).tobytes() == X.tobytes()


def test_bvecs_widening_and_mismatch(tmp_path):
    p = tmp_path / "one.bvecs"
    p.write_bytes(struct.pack("<i", 3) + bytes([0, 128, 255]))
    X = read_bvecs(p)
    assert X.dtype == np.float32
    np.testing.assert_array_equal(X, [[0.0, 128.0, 255.0]])
    q = tmp_path / "mixed.bvecs"
    q.write_bytes(struct.pack("<i", 2) + b"\x00\x01" + struct.pack("<i", 4) + b"\x00\x01\x02\x03")
    with pytest.raises(FormatError, match="2 and 4"):
        read_bvecs(q)
    z = tmp_path / "zero.bvecs"
    z.write_bytes(struct.pack("<i", 0))
    with pytest.raises(FormatError):
        read_bvecs(z)


def test_ivecs_bytes_empty_round_trip(tmp_path):
    p = tmp_path / "gt.ivecs"
    write_ivecs(p, [[5, 7]])
    assert p.read_bytes() == bytes.fromhex("02000000" "05000000" "07000000")
    e = tmp_path / "empty.ivecs"
    write_ivecs(e, [])
    assert e.read_bytes() == b"" and read_ivecs(e).size == 0
    rows = np.random.default_rng(3).integers(-(2**31), 2**31 - 1, size=(9, 4))
    r = tmp_path / "rt.ivecs"
    write_ivecs(r, rows)
    np.testing.assert_array_equal(read_ivecs(r), rows)
    with pytest.raises(ValueError):
        write_ivecs(tmp_path / "x.ivecs", np.array([[1], [2, 3]], dtype=object))
    with pytest.raises(ValueError):
        write_ivecs(tmp_path / "y.ivecs", [[2**31]])


def test_vecsfile_chunked_header_check(tmp_path):
    """A mid-file dimension switch in a file with no trailing bytes is found by the
    chunk that holds it, with the reference's message and byte offset."""
    d, n = 4, 10
    raw = bytearray()
    for i in range(n):
        raw += struct.pack("<i", d if i != 7 else 5) + bytes(range(i, i + d))
    p = tmp_path / "sw.bvecs"
    p.write_bytes(bytes(raw))
    f = VecsFile(p)
    assert (f.n, f.d, f.kind, f.record_bytes) == (n, d, "bvecs", 8)
    np.testing.assert_array_equal(f.rows(0, 3)[2], [2, 3, 4, 5])
    f.check_headers(0, 7)
    with pytest.raises(FormatError, match="inconsistent dimensions 4 and 5 at byte offset 56"):
        f.rows(4, 10)
    with pytest.raises(FormatError, match="inconsistent dimensions 4 and 5 at byte offset 56"):
        read_bvecs(p)
    with pytest.raises(ValueError, match="record kind"):
        VecsFile(tmp_path / "x.dat")


def test_encoded_writer_streams_same_bytes(tmp_path):
    rng = np.random.default_rng(1)
    codes = rng.integers(0, 256, size=(1000, 8)).astype(np.uint8)
    whole, streamed = tmp_path / "a.hcle", tmp_path / "b.hcle"
    write_encoded(whole, EncodedDataset(codes=codes, k_count=256))
    with EncodedWriter(streamed, 1000, 8, 256) as w:
        for r0 in range(0, 1000, 300):
            w.write(codes[r0:r0 + 300])
    assert whole.read_bytes() == streamed.read_bytes()
    m = read_encoded(streamed, mmap=True)
    assert isinstance(m.codes, np.ndarray)
    np.testing.assert_array_equal(m.codes, codes)
    np.testing.assert_array_equal(read_encoded(streamed).codes, codes)
    # wide codes (K > 256)
    wide = rng.integers(0, 300, size=(5, 3)).astype(np.uint16)
    with EncodedWriter(tmp_path / "w.hcle", 5, 3, 300) as w:
        w.write(wide)
    np.testing.assert_array_equal(read_encoded(tmp_path / "w.hcle", mmap=True).codes, wide)
    # short write and abort
    w = EncodedWriter(tmp_path / "short.hcle", 4, 2, 16)
    w.write(np.zeros((3, 2), np.uint8))
    with pytest.raises(ValueError, match="3 rows written"):
        w.close()
    with pytest.raises(ZeroDivisionError):
        with EncodedWriter(tmp_path / "gone.hcle", 1, 1, 4):
            1 / 0
    assert not (tmp_path / "gone.hcle").exists()
    t = tmp_path / "trunc.hcle"
    t.write_bytes(streamed.read_bytes()[:-1])
    with pytest.raises(FormatError, match="truncated"):
        read_encoded(t, mmap=True)
