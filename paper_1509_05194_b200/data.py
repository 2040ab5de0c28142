"""Dataset ingestion at 1e9 scale (reference annq/data.py:50-165).

Same on-disk formats and the same public readers/writers as the reference
(texmex records: a little-endian int32 dimension header, then d float32 values
for fvecs, d bytes for bvecs, d int32 values for ivecs; every record of a file
has the same d), with the same FormatError messages and byte offsets.

What is new is the streaming path for files that do not fit host memory:

* :class:`VecsFile` memory-maps a file, validates its layout from the size and
  the first header, and hands out raw record rows (headers checked per chunk);
* :func:`encode_vecs` beam-encodes a whole fvecs/bvecs file on the GPU: raw
  record bytes stream through pinned slots (a worker thread copies and
  validates them), are uploaded as they lie in the file (one byte per bvecs
  value on the bus) and unpacked on the device by ``da_unpack_vecs``, then
  encoded; codes land in an :class:`~.codebook.EncodedDataset` or straight in an
  HCLE file (:class:`~.codebook.EncodedWriter`).

The readers are host I/O (file parsing, no arithmetic); the encode path has no
CPU fallback.
"""

from __future__ import annotations

import os

import numpy as np

from .groundtruth import GroundTruth, brute_force_knn
from .validation import FormatError, check_vectors

__all__ = ["GroundTruth", "VecsFile", "brute_force_knn", "encode_vecs", "read_bvecs", "read_fvecs", "read_ivecs",
           "write_fvecs", "write_ivecs"]

_VALUE_BYTES = {"fvecs": 4, "ivecs": 4, "bvecs": 1}


def _kind_of(path, kind):
    if kind is not None:
        if kind not in _VALUE_BYTES:
            raise ValueError(f"unknown record kind {kind!r} (fvecs, bvecs or ivecs)")
        return kind
    ext = os.path.splitext(str(path))[1].lstrip(".").lower()
    if ext not in _VALUE_BYTES:
        raise ValueError(f"{path}: cannot infer the record kind from the extension; pass kind=")
    return ext


class VecsFile:
    """Memory-mapped texmex record file.

    The layout checks of the reference parser (data.py:50-91) run up front on the
    file size and the first and last headers; the headers of full records are
    checked chunk by chunk as rows are read (:meth:`rows`), so a mid-file
    dimension switch raises the same FormatError when its chunk is reached.
    """

    def __init__(self, path, kind: str | None = None):
        self.path = path
        self.kind = _kind_of(path, kind)
        vb = _VALUE_BYTES[self.kind]
        size = os.path.getsize(path)
        self.size = size
        if size == 0:
            self.n, self.d, self.record_bytes, self._map = 0, 0, 0, None
            return
        if size < 4:
            raise FormatError(f"{path}: truncated record header at byte offset 0")
        self._map = np.memmap(path, dtype=np.uint8, mode="r")
        d = int(self._map[:4].view("<i4")[0])
        if d <= 0:
            raise FormatError(f"{path}: invalid dimension header {d} at byte offset 0")
        rec = 4 + d * vb
        n = size // rec
        tail = size - n * rec
        self.n, self.d, self.record_bytes = n, d, rec
        if tail:
            # the reference names a mid-file switch before the trailing bytes
            self.check_headers(0, n)
            base = n * rec
            if tail < 4:
                raise FormatError(f"{path}: truncated record header at byte offset {base}")
            d_last = int(self._map[base:base + 4].view("<i4")[0])
            if d_last != d:
                raise FormatError(f"{path}: inconsistent dimensions {d} and {d_last} at byte offset {base}")
            raise FormatError(f"{path}: truncated record at byte offset {base + 4}")

    def raw(self, r0: int, r1: int) -> np.ndarray:
        """(r1 - r0, record_bytes) uint8 view of records [r0, r1), headers unchecked."""
        if self._map is None:
            return np.empty((0, 0), dtype=np.uint8)
        rec = self.record_bytes
        return self._map[r0 * rec:r1 * rec].reshape(r1 - r0, rec)

    def check_headers(self, r0: int, r1: int, raw: np.ndarray | None = None) -> None:
        """Every header of records [r0, r1) equals d (FormatError with the byte offset)."""
        if r1 <= r0:
            return
        rows = self.raw(r0, r1) if raw is None else raw
        heads = np.ascontiguousarray(rows[:, :4]).view("<i4").ravel()
        bad = np.flatnonzero(heads != self.d)
        if bad.size:
            i = r0 + int(bad[0])
            raise FormatError(f"{self.path}: inconsistent dimensions {self.d} and {int(heads[bad[0]])} "
                              f"at byte offset {i * self.record_bytes}")

    def rows(self, r0: int, r1: int) -> np.ndarray:
        """Payload of records [r0, r1) as stored (float32 / uint8 / int32), headers checked."""
        self.check_headers(r0, r1)
        raw = self.raw(r0, r1)
        dt = {"fvecs": "<f4", "bvecs": np.uint8, "ivecs": "<i4"}[self.kind]
        return raw[:, 4:].view(dt) if self.kind != "bvecs" else raw[:, 4:]


def read_fvecs(path) -> np.ndarray:
    """(n, d) float32, bit-exact; an empty file gives a (0, 0) array (data.py:94-107)."""
    f = VecsFile(path, "fvecs")
    if f.n == 0:
        return np.empty((0, 0), dtype=np.float32)
    out = np.ascontiguousarray(f.rows(0, f.n), dtype=np.float32)
    if not np.isfinite(out).all():
        raise FormatError(f"{path}: non-finite value in payload")
    return out


def read_bvecs(path) -> np.ndarray:
    """(n, d) float32 widened exactly from unsigned bytes (data.py:126-134)."""
    f = VecsFile(path, "bvecs")
    if f.n == 0:
        return np.empty((0, 0), dtype=np.float32)
    return f.rows(0, f.n).astype(np.float32)


def read_ivecs(path) -> np.ndarray:
    """(n, d) int64 (data.py:137-145)."""
    f = VecsFile(path, "ivecs")
    if f.n == 0:
        return np.empty((0, 0), dtype=np.int64)
    return f.rows(0, f.n).astype(np.int64)


def _write_records(path, payload: np.ndarray, head_dtype) -> None:
    n, d = payload.shape
    with open(path, "wb") as fh:
        if n == 0:
            return
        rec = np.empty((n, d + 1), dtype=head_dtype)
        rec.view("<i4")[:, 0] = d
        rec[:, 1:] = payload
        fh.write(rec.tobytes())


def write_fvecs(path, X) -> None:
    """(n, d) floats as fvecs; read_fvecs round-trips it (data.py:110-123)."""
    X = check_vectors(X, name="X", allow_empty=True)
    _write_records(path, X, "<f4")


def write_ivecs(path, rows) -> None:
    """Rectangular integer rows as ivecs, int32 range enforced (data.py:148-165)."""
    rows = np.asarray(rows)
    if rows.ndim == 1 and rows.size == 0:
        rows = rows.reshape(0, 0)
    if rows.ndim != 2:
        raise ValueError(f"rows must be rectangular 2-D, got shape {rows.shape}")
    info = np.iinfo(np.int32)
    if rows.size and (rows.min() < info.min or rows.max() > info.max):
        raise ValueError("rows contain values outside the i32 range")
    try:
        _write_records(path, rows, "<i4")
    except OSError as e:
        raise OSError(f"failed writing {path}: {e}") from e


def encode_vecs(codebook, path, beam_width: int = 10, *, out_path=None, kind: str | None = None,
                cross=None, chunk_rows: int = 1 << 18):
    """Beam-encode every record of an fvecs/bvecs file on the GPU, streamed.

    Returns the :class:`~.codebook.EncodedDataset` (codes identical to
    ``encode_dataset(codebook, read_bvecs(path), beam_width)``).  With
    ``out_path`` the codes are also written as an HCLE file chunk by chunk and
    the returned dataset's codes are a read-only memory map of that file, so
    host memory stays bounded at 1e9 vectors.
    """
    from . import _engine as E
    from .codebook import EncodedDataset, EncodedWriter, _codebook_dev, _cross_dev, _torch_code_dtype, \
        cross_products

    if beam_width < 1:
        raise ValueError("beam_width must be >= 1")
    f = VecsFile(path, kind)
    if f.kind == "ivecs":
        raise ValueError(f"{path}: ivecs holds ids, not vectors")
    if f.n and f.d != codebook.dim:
        raise ValueError(f"data d={f.d} does not match codebook dim {codebook.dim}")
    M, K = codebook.m_count, codebook.k_count
    writer = EncodedWriter(out_path, f.n, M, K) if out_path is not None else None
    if f.n == 0:
        codes = np.empty((0, M), dtype=codebook.code_dtype)
        if writer is not None:
            writer.close()
        return EncodedDataset(codes=codes, k_count=K, codebook_hash=codebook.content_hash())
    if cross is None:
        cross = cross_products(codebook)
    cw, sq = _codebook_dev(codebook)
    Pt, _ = _cross_dev(cross)

    def fill(slot, r0, rows):
        raw = f.raw(r0, r0 + rows)
        f.check_headers(r0, r0 + rows, raw)
        np.copyto(slot[: rows * f.record_bytes].numpy().reshape(rows, f.record_bytes), raw)

    codes_dev, bad = E.encode_records(fill, f.n, f.d, 1 if f.kind == "bvecs" else 0, cw, sq, Pt, beam_width,
                                      out_dtype=_torch_code_dtype(K), chunk=chunk_rows)
    if bad:
        if writer is not None:
            writer.abort()
        raise FormatError(f"{path}: non-finite value in payload")
    if writer is None:
        codes = codes_dev.cpu().numpy()
    else:
        step = max(1, (1 << 26) // max(M, 1))
        for r0 in range(0, f.n, step):
            writer.write(codes_dev[r0:r0 + step].cpu().numpy())
        writer.close()
        codes = writer.codes_map()
    return EncodedDataset(codes=codes, k_count=K, codebook_hash=codebook.content_hash())
