"""Streamed file encode: encode_vecs over fvecs/bvecs files
returns exactly encode_dataset(read_*(path)) and, with out_path, writes the same
HCLE bytes as write_encoded; payload and header errors surface as FormatError."""

import struct

import numpy as np
import pytest

import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import FormatError, synthetic
from paper_1509_05194_b200.data import encode_vecs, read_bvecs, read_fvecs, write_fvecs

pytestmark = pytest.mark.gpu


def _book(D, M=4, K=64, seed=0):
    rng = np.random.default_rng(seed)
    return da.Codebook(codewords=(rng.standard_normal((M, K, D)) * 20).astype(np.float32), order=np.arange(M))


def _write_bvecs(path, U8):
    n, d = U8.shape
    rec = np.empty((n, 4 + d), dtype=np.uint8)
    rec[:, :4] = np.frombuffer(struct.pack("<i", d), dtype=np.uint8)
    rec[:, 4:] = U8
    path.write_bytes(rec.tobytes())


@pytest.mark.parametrize("chunk", [64, 1000, 1 << 18])
def test_bvecs_stream_matches_encode_dataset(tmp_path, chunk):
    X = synthetic.config_b(n=3001, seed=5, chunk=3001)        # integers in [0, 255]
    p = tmp_path / "x.bvecs"
    _write_bvecs(p, X.astype(np.uint8))
    book = _book(128, M=8, K=256)
    ref = da.encode_dataset(book, read_bvecs(p), beam_width=10)
    got = encode_vecs(book, p, beam_width=10, chunk_rows=chunk)
    np.testing.assert_array_equal(got.codes, ref.codes)
    assert got.codebook_hash == book.content_hash()
    out = tmp_path / "x.hcle"
    got2 = encode_vecs(book, p, beam_width=10, out_path=out, chunk_rows=chunk)
    np.testing.assert_array_equal(got2.codes, ref.codes)
    whole = tmp_path / "w.hcle"
    da.write_encoded(whole, ref)
    assert out.read_bytes() == whole.read_bytes()


def test_fvecs_stream_and_errors(tmp_path):
    rng = np.random.default_rng(2)
    X = rng.standard_normal((777, 12)).astype(np.float32) * 3
    p = tmp_path / "x.fvecs"
    write_fvecs(p, X)
    book = _book(12)
    for L in (1, 4):
        np.testing.assert_array_equal(encode_vecs(book, p, L, chunk_rows=100).codes,
                                      da.encode_dataset(book, read_fvecs(p), L).codes)
    # non-finite payload: FormatError like read_fvecs, and no partial HCLE left behind
    Y = X.copy()
    Y[500, 3] = np.inf
    raw = bytearray(p.read_bytes())
    off = 500 * (4 + 48) + 4 + 3 * 4
    raw[off:off + 4] = struct.pack("<f", float("inf"))
    q = tmp_path / "inf.fvecs"
    q.write_bytes(bytes(raw))
    with pytest.raises(FormatError, match="non-finite value in payload"):
        encode_vecs(book, q, 4, out_path=tmp_path / "inf.hcle", chunk_rows=128)
    assert not (tmp_path / "inf.hcle").exists()
    # a dimension switch in a later chunk
    raw = bytearray(p.read_bytes())
    raw[600 * 52:600 * 52 + 4] = struct.pack("<i", 13)
    s = tmp_path / "sw.fvecs"
    s.write_bytes(bytes(raw))
    with pytest.raises(FormatError, match=f"inconsistent dimensions 12 and 13 at byte offset {600 * 52}"):
        encode_vecs(book, s, 4, chunk_rows=128)
    # empty file and dimension mismatch
    e = tmp_path / "e.fvecs"
    e.write_bytes(b"")
    assert encode_vecs(book, e, 4).codes.shape == (0, 4)
    with pytest.raises(ValueError, match="does not match codebook dim"):
        encode_vecs(_book(13), p, 4)
