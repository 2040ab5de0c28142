"""Additive codebook model, beam-search encoding and ADC on the B200.

Drop-in for annq/codebook.py (same names, signatures, dtypes and errors).
Host objects keep the reference's fields (numpy arrays); the arithmetic runs
in the CUDA kernels of libda_b200 (include/da_b200.h).  Each object caches
its device copy so repeated calls do not re-upload.

Reference map (annq/codebook.py):
  Codebook :62-132   CrossProductTable :135-140   EncodedDataset :143-166
  AdcTable :169-174  reconstruct :191-195         distortion :198-208
  dictionary_variances / reorder_by_variance :211-228
  cross_products / refresh_cross_products :231-252
  encode_multipath :303-316   encode_dataset :319-358
  adc_table :361-369  adc_distance :372-385  code_pair_sums :388-396
  exhaustive_adc_search :399-429
"""

from __future__ import annotations

import hashlib
import os
import struct
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _engine as E
from .validation import FormatError, check_codes, check_query, check_vectors

__all__ = [
    "Codebook",
    "CrossProductTable",
    "EncodedDataset",
    "EncodedWriter",
    "AdcTable",
    "reconstruct",
    "distortion",
    "dictionary_variances",
    "reorder_by_variance",
    "cross_products",
    "refresh_cross_products",
    "encode_multipath",
    "encode_dataset",
    "adc_table",
    "adc_distance",
    "code_pair_sums",
    "exhaustive_adc_search",
    "exhaustive_adc_search_batch",
    "adc_rerank",
    "write_codebook",
    "read_codebook",
    "write_encoded",
    "read_encoded",
]

CODEBOOK_MAGIC = b"HCLB"
ENCODED_MAGIC = b"HCLE"
FORMAT_VERSION = 1
MAX_CODEWORDS = 65536

# Same contract as the reference (codebook.py:53-55): one count per kernel
# that reads raw d-dimensional vectors.  An encode call reads them twice
# (score-table build, final exact error); the beam stages read tables only.
DEBUG_COUNTERS = {"raw_dim_kernel_calls": 0}


def _raw_kernel(n=1):
    DEBUG_COUNTERS["raw_dim_kernel_calls"] += n


def _code_dtype(k_count: int):
    return np.uint8 if k_count <= 256 else np.uint16


def _torch_code_dtype(k_count: int):
    return torch.uint8 if k_count <= 256 else torch.uint16


@dataclass
class Codebook:
    """M x K x d additive codebook; ``order[j]`` = source slot of dictionary j."""

    codewords: np.ndarray  # (M, K, d) float32
    order: np.ndarray      # (M,) int64

    def __post_init__(self):
        self.codewords = np.ascontiguousarray(self.codewords, dtype=np.float32)
        if self.codewords.ndim != 3:
            raise ValueError("codewords must have shape (M, K, d)")
        if self.k_count > MAX_CODEWORDS:
            raise ValueError(f"K={self.k_count} exceeds the supported maximum {MAX_CODEWORDS}")
        self.order = np.asarray(self.order, dtype=np.int64)
        if self.order.shape != (self.m_count,):
            raise ValueError("order must be a permutation of length M")

    @classmethod
    def zeros(cls, m_count, k_count, dim) -> "Codebook":
        return cls(codewords=np.zeros((m_count, k_count, dim), dtype=np.float32),
                   order=np.arange(m_count, dtype=np.int64))

    @property
    def m_count(self) -> int:
        return self.codewords.shape[0]

    @property
    def k_count(self) -> int:
        return self.codewords.shape[1]

    @property
    def dim(self) -> int:
        return self.codewords.shape[2]

    @property
    def code_dtype(self):
        return _code_dtype(self.k_count)

    def content_hash(self) -> bytes:
        """sha256 over (<III d, M, K) + float32 codewords + order as <u4."""
        cached = self.__dict__.get("_hash_cache")
        if cached is None:
            h = hashlib.sha256()
            h.update(struct.pack("<III", self.dim, self.m_count, self.k_count))
            h.update(np.ascontiguousarray(self.codewords, dtype="<f4").tobytes())
            h.update(self.order.astype("<u4").tobytes())
            cached = h.digest()
            self.__dict__["_hash_cache"] = cached
        return cached


def _codebook_dev(codebook):
    """(cw float32 (M,K,D), sq float64 (M,K)) on the current device, cached."""
    dev = E.device()
    cache = getattr(codebook, "__dict__", {}).get("_dev_cache")
    cw_np = codebook.codewords
    if cache is not None and cache[0] is cw_np and cache[1] == dev:
        return cache[2], cache[3]
    cw = E.to_dev(np.ascontiguousarray(cw_np, dtype=np.float32))
    sq = E.einsum_sq(cw)
    try:
        codebook.__dict__["_dev_cache"] = (cw_np, dev, cw, sq)
    except (AttributeError, TypeError):
        pass
    return cw, sq


class CrossProductTable:
    """products[a, b][i, j] = c_a(i).c_b(j) (M,M,K,K) f64 plus sq_norms (M,K) f64.

    Device-resident; the host arrays are materialised on first access.
    """

    def __init__(self, products=None, sq_norms=None):
        self._products = None if products is None else np.asarray(products, dtype=np.float64)
        self._sq = None if sq_norms is None else np.asarray(sq_norms, dtype=np.float64)
        self._dev = None

    @classmethod
    def _from_device(cls, Pt: torch.Tensor, sq: torch.Tensor) -> "CrossProductTable":
        t = cls()
        t._dev = (Pt.device, Pt, sq)
        return t

    @property
    def products(self) -> np.ndarray:
        if self._products is None:
            self._products = self._dev[1].cpu().numpy()
        return self._products

    @property
    def sq_norms(self) -> np.ndarray:
        if self._sq is None:
            self._sq = self._dev[2].cpu().numpy()
        return self._sq

    def device(self):
        dev = E.device()
        if self._dev is not None and self._dev[0] == dev:
            return self._dev[1], self._dev[2]
        Pt = E.to_dev(np.ascontiguousarray(self.products, dtype=np.float64))
        sq = E.to_dev(np.ascontiguousarray(self.sq_norms, dtype=np.float64))
        self._dev = (dev, Pt, sq)
        return Pt, sq

    def __repr__(self):
        shape = tuple(self._dev[1].shape) if self._dev is not None else np.shape(self._products)
        return f"CrossProductTable(shape={shape})"


_foreign = {}


def _cross_dev(cross):
    """Device tables for our CrossProductTable or any object with .products/.sq_norms."""
    if isinstance(cross, CrossProductTable):
        return cross.device()
    key = id(cross)
    hit = _foreign.get(key)
    if hit is not None and hit[0]() is cross:
        return hit[1], hit[2]
    Pt = E.to_dev(np.ascontiguousarray(cross.products, dtype=np.float64))
    sq = E.to_dev(np.ascontiguousarray(cross.sq_norms, dtype=np.float64))
    try:
        _foreign[key] = (weakref.ref(cross), Pt, sq)
    except TypeError:
        pass
    if len(_foreign) > 8:
        _foreign.pop(next(iter(_foreign)))
    return Pt, sq


@dataclass
class EncodedDataset:
    """n x M code matrix (uint8 if K <= 256 else uint16), optional int64 id_map."""

    codes: np.ndarray
    k_count: int
    codebook_hash: bytes | None = None
    id_map: np.ndarray | None = None

    def __post_init__(self):
        check_codes(self.codes, self.k_count, name="codes")
        self.codes = np.ascontiguousarray(self.codes, dtype=_code_dtype(self.k_count))
        if self.id_map is not None:
            self.id_map = np.asarray(self.id_map, dtype=np.int64)
            if self.id_map.shape != (self.n,):
                raise ValueError("id_map length must match the number of codes")

    @property
    def n(self) -> int:
        return self.codes.shape[0]

    @property
    def m_count(self) -> int:
        return self.codes.shape[1]


def _encoded_dev(encoded):
    cache = getattr(encoded, "__dict__", {}).get("_dev_cache")
    dev = E.device()
    if cache is not None and cache[0] is encoded.codes and cache[1] == dev:
        return cache[2]
    t = E.to_dev(np.ascontiguousarray(encoded.codes))
    try:
        encoded.__dict__["_dev_cache"] = (encoded.codes, dev, t)
    except (AttributeError, TypeError):
        pass
    return t


@dataclass(frozen=True)
class AdcTable:
    """values[m, k] = ||q - c_m(k)||^2 (clipped at 0), plus ||q||^2."""

    values: np.ndarray
    q_sq_norm: float


# ---------------------------------------------------------------------------


def reconstruct(codebook: Codebook, code) -> np.ndarray:
    """sum_m c_m(code_m) as (d,) float64."""
    code = check_codes(np.asarray(code).reshape(1, -1), codebook.k_count, m_count=codebook.m_count, name="code")
    _raw_kernel()
    cw, _ = _codebook_dev(codebook)
    codes = E.to_dev(code.astype(np.int32))
    return E.reconstruct(codes, cw)[0].cpu().numpy()


def distortion(codebook: Codebook, data, encoded: EncodedDataset) -> float:
    """Mean squared reconstruction error of data under its codes."""
    X = check_vectors(data, name="data")
    if encoded.n != X.shape[0]:
        raise ValueError(f"codes cover {encoded.n} vectors, data has {X.shape[0]}")
    if X.shape[1] != codebook.dim:
        raise ValueError(f"data d={X.shape[1]} does not match codebook dim {codebook.dim}")
    codes = check_codes(encoded.codes, codebook.k_count, m_count=codebook.m_count)
    _raw_kernel()
    cw, _ = _codebook_dev(codebook)
    Xd = E.to_dev(X)
    cd = E.to_dev(np.ascontiguousarray(codes.astype(np.int32)))
    return float(E.np_mean(E.vec_err(Xd, cd, cw)).item())


def dictionary_variances(codebook: Codebook) -> np.ndarray:
    """Per-dictionary mean squared distance of codewords to their mean (host, M*K*d)."""
    cw = codebook.codewords.astype(np.float64)
    centered = cw - cw.mean(axis=1, keepdims=True)
    return (centered * centered).sum(axis=2).mean(axis=1)


def reorder_by_variance(codebook: Codebook):
    """(codebook with dictionaries in non-increasing variance, permutation)."""
    perm = np.argsort(-dictionary_variances(codebook), kind="stable").astype(np.int64)
    return Codebook(codewords=codebook.codewords[perm].copy(), order=codebook.order[perm].copy()), perm


def cross_products(codebook: Codebook) -> CrossProductTable:
    """All pairwise codeword inner products (device GEMM)."""
    cw, _ = _codebook_dev(codebook)
    Pt, sq = E.cross_full(cw)
    return CrossProductTable._from_device(Pt, sq)


def refresh_cross_products(cross, codebook: Codebook, m: int) -> CrossProductTable:
    """Fresh table equal to `cross` with the rows/cols of dictionary m rebuilt."""
    cw, _ = _codebook_dev(codebook)
    Pt0, sq0 = _cross_dev(cross)
    Pt, sq = Pt0.clone(), sq0.clone()
    E.cross_refresh(cw, m, Pt, sq)
    return CrossProductTable._from_device(Pt, sq)


def encode_multipath(codebook: Codebook, cross, x, beam_width: int):
    """Encode one vector with beam width L -> (code, exact squared error)."""
    if beam_width < 1:
        raise ValueError("beam_width must be >= 1")
    x = check_query(x, codebook.dim, name="x")
    _raw_kernel(2)
    cw, sq = _codebook_dev(codebook)
    Pt, _ = _cross_dev(cross)
    Xd = E.to_dev(x.reshape(1, -1))
    codes, err = E.encode(Xd, cw, sq, Pt, beam_width, out_dtype=torch.int32)
    return codes[0].cpu().numpy().astype(codebook.code_dtype), float(err[0].item())


def encode_dataset(codebook: Codebook, data, beam_width: int = 10, n_jobs: int = 1,
                   cross=None) -> EncodedDataset:
    """Beam-encode every vector; byte-identical for any n_jobs (ignored on the GPU)."""
    if beam_width < 1:
        raise ValueError("beam_width must be >= 1")
    X = check_vectors(data, name="data", allow_empty=True, finite=False)
    if X.shape[0] and X.shape[1] != codebook.dim:
        raise ValueError(f"data d={X.shape[1]} does not match codebook dim {codebook.dim}")
    if X.shape[0] == 0:
        return EncodedDataset(codes=np.empty((0, codebook.m_count), dtype=codebook.code_dtype),
                              k_count=codebook.k_count, codebook_hash=codebook.content_hash())
    if cross is None:
        cross = cross_products(codebook)
    _raw_kernel(2)
    cw, sq = _codebook_dev(codebook)
    Pt, _ = _cross_dev(cross)
    # host rows stream through pinned buffers: upload, finiteness check and encode overlap
    codes = E.encode_host(X, cw, sq, Pt, beam_width, out_dtype=_torch_code_dtype(codebook.k_count))
    return EncodedDataset(codes=codes.cpu().numpy(), k_count=codebook.k_count,
                          codebook_hash=codebook.content_hash())


def adc_table(codebook: Codebook, q) -> AdcTable:
    """values[m, k] = ||q - c_m(k)||^2 for one query (device GEMV + clip)."""
    q = check_query(q, codebook.dim)
    _raw_kernel()
    cw, sq = _codebook_dev(codebook)
    lut, qsq = E.adc_lut(E.to_dev(q.reshape(1, -1)), cw, sq)
    return AdcTable(values=lut[0].cpu().numpy(), q_sq_norm=float(qsq[0].item()))


def adc_distance(table: AdcTable, cross, code) -> float:
    """||q - sum_m c_m||^2 for ONE code from its table (scalar host bookkeeping)."""
    code = np.asarray(code, dtype=np.int64).reshape(-1)
    M = table.values.shape[0]
    total = float(table.values[np.arange(M), code].sum())
    total -= (M - 1) * table.q_sq_norm
    prods = cross.products
    for a in range(M):
        for b in range(a + 1, M):
            total += 2.0 * float(prods[a, b][code[a], code[b]])
    return total


def code_pair_sums(cross, codes) -> np.ndarray:
    """2 * sum_{a<b} P[a,b][i_a, i_b] per code row (device gather)."""
    codes = np.asarray(codes, dtype=np.int64)
    if codes.ndim != 2:
        raise ValueError("codes must be 2-D (n, M)")
    if codes.shape[0] == 0:
        return np.zeros(0)
    Pt, _ = _cross_dev(cross)
    cd = E.to_dev(np.ascontiguousarray(codes.astype(np.int32)))
    return E.pair_sums(cd, Pt).cpu().numpy()


def _search_inputs(codebook, encoded, cross, pair_sums):
    if cross is None:
        cross = cross_products(codebook)
    Pt, _ = _cross_dev(cross)
    codes_d = _encoded_dev(encoded)
    if pair_sums is None:
        pair_d = E.pair_sums(codes_d, Pt)
    else:
        pair_d = E.to_dev(np.ascontiguousarray(pair_sums, dtype=np.float64))
    return codes_d, pair_d


def _scan(codebook, encoded, cross, pair_sums, lut, qsq, r, cand=None):
    """Top-r ADC scan: packed 16-byte records (codes + pair sum, one sector per
    random candidate) when the codes fit, else the generic kernel."""
    packed = None
    cache = getattr(encoded, "__dict__", {}).get("_packed_cache")
    dev = E.device()
    if pair_sums is None and cache is not None and cache[0] is encoded.codes and cache[1] is cross and cache[2] == dev:
        packed = cache[3]
    if packed is None:
        codes_d, pair_d = _search_inputs(codebook, encoded, cross, pair_sums)
        packed = E.adc_pack(codes_d, pair_d)
        if packed is None:
            return E.adc_scan(codes_d, pair_d, lut, qsq, r, cand=cand)
        if pair_sums is None and cross is not None:
            try:
                encoded.__dict__["_packed_cache"] = (encoded.codes, cross, dev, packed)
            except (AttributeError, TypeError):
                pass
    return E.adc_scan_packed(packed, lut, qsq, r, cand=cand)


def exhaustive_adc_search(codebook: Codebook, encoded: EncodedDataset, q, r: int, cross=None,
                          pair_sums: np.ndarray | None = None):
    """Exact top-r under adc_distance, ties by lower position -> (ids int64, dists f64)."""
    if r < 1 or r > encoded.n:
        raise ValueError(f"r={r} must be in [1, {encoded.n}]")
    q = check_query(q, codebook.dim)
    ids, d = exhaustive_adc_search_batch(codebook, encoded, q.reshape(1, -1), r, cross, pair_sums)
    return ids[0], d[0]


def exhaustive_adc_search_batch(codebook: Codebook, encoded: EncodedDataset, Q, r: int, cross=None,
                                pair_sums: np.ndarray | None = None):
    """Batched exhaustive_adc_search: Q (nq, d) -> ids (nq, r) int64, dists (nq, r) f64."""
    if r < 1 or r > encoded.n:
        raise ValueError(f"r={r} must be in [1, {encoded.n}]")
    Q = np.asarray(Q, dtype=np.float64)
    if Q.ndim != 2 or Q.shape[1] != codebook.dim:
        raise ValueError(f"queries must be (nq, {codebook.dim})")
    if not np.isfinite(Q).all():
        raise ValueError("queries contain non-finite values")
    _raw_kernel()
    cw, sq = _codebook_dev(codebook)
    lut, qsq = E.adc_lut(E.to_dev(Q), cw, sq)
    ids, dists = _scan(codebook, encoded, cross, pair_sums, lut, qsq, r)
    ids = ids.cpu().numpy()
    if encoded.id_map is not None:
        ids = encoded.id_map[ids]
    return ids.astype(np.int64), dists.cpu().numpy()


def adc_rerank(codebook: Codebook, encoded: EncodedDataset, Q, candidates, r: int, cross=None,
               pair_sums: np.ndarray | None = None):
    """Score per-query candidate row lists (nq, ncand) and keep the top r of each.

    Same semantics as exhaustive_adc_search on EncodedDataset(codes[cand],
    id_map=cand) with pair_sums[cand]: ties by position in the list.
    """
    cand = np.ascontiguousarray(candidates, dtype=np.int64)
    Q = np.asarray(Q, dtype=np.float64)
    if cand.ndim != 2 or Q.ndim != 2 or cand.shape[0] != Q.shape[0]:
        raise ValueError("candidates must be (nq, ncand) and queries (nq, d)")
    if r < 1 or r > cand.shape[1]:
        raise ValueError(f"r={r} must be in [1, {cand.shape[1]}]")
    if cand.size and (cand.min() < 0 or cand.max() >= encoded.n):
        raise ValueError("candidate ids outside the encoded set")
    cw, sq = _codebook_dev(codebook)
    lut, qsq = E.adc_lut(E.to_dev(Q), cw, sq)
    ids, dists = _scan(codebook, encoded, cross, pair_sums, lut, qsq, r, cand=E.to_dev(cand))
    ids = ids.cpu().numpy()
    if encoded.id_map is not None:
        ids = encoded.id_map[ids]
    return ids.astype(np.int64), dists.cpu().numpy()


# ---------------------------------------------------------------------------
# file formats (host I/O, unchanged from codebook.py:443-494 so checkpoints
# written by either implementation load in the other)


def _read_exact(f, count, path, what):
    buf = f.read(count)
    if len(buf) != count:
        raise FormatError(f"{path}: truncated while reading {what}")
    return buf


def write_codebook(path, codebook: Codebook) -> None:
    with open(path, "wb") as f:
        f.write(CODEBOOK_MAGIC)
        f.write(struct.pack("<IIII", FORMAT_VERSION, codebook.dim, codebook.m_count, codebook.k_count))
        f.write(np.ascontiguousarray(codebook.codewords, dtype="<f4").tobytes())
        f.write(codebook.order.astype("<u4").tobytes())


def read_codebook(path) -> Codebook:
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != CODEBOOK_MAGIC:
            raise FormatError(f"{path}: bad magic {magic!r}, expected {CODEBOOK_MAGIC!r}", exit_code=2)
        version, d, M, K = struct.unpack("<IIII", _read_exact(f, 16, path, "header"))
        if version != FORMAT_VERSION:
            raise FormatError(f"{path}: unsupported format version {version}")
        cw = np.frombuffer(_read_exact(f, 4 * M * K * d, path, "codewords"), dtype="<f4")
        order = np.frombuffer(_read_exact(f, 4 * M, path, "order"), dtype="<u4")
        return Codebook(codewords=cw.reshape(M, K, d).copy(), order=order.astype(np.int64))


def write_encoded(path, encoded: EncodedDataset) -> None:
    width = 1 if encoded.k_count <= 256 else 2
    with open(path, "wb") as f:
        f.write(ENCODED_MAGIC)
        f.write(struct.pack("<IQIIB", FORMAT_VERSION, encoded.n, encoded.m_count, encoded.k_count, width))
        f.write(np.ascontiguousarray(encoded.codes, dtype=f"<u{width}").tobytes())


_ENCODED_HEADER = 4 + struct.calcsize("<IQIIB")


class EncodedWriter:
    """HCLE file written chunk by chunk (same bytes as write_encoded of the whole
    set): header first, then codes in row order.  For code sets that never sit
    in host memory at once (1e9 rows = 8 GB of uint8 codes)."""

    def __init__(self, path, n: int, m_count: int, k_count: int):
        self.path, self.n, self.m_count, self.k_count = path, int(n), int(m_count), int(k_count)
        self.width = 1 if k_count <= 256 else 2
        self.rows = 0
        self._f = open(path, "wb")
        self._f.write(ENCODED_MAGIC)
        self._f.write(struct.pack("<IQIIB", FORMAT_VERSION, self.n, self.m_count, self.k_count, self.width))

    def write(self, codes) -> None:
        codes = np.asarray(codes)
        if codes.ndim != 2 or codes.shape[1] != self.m_count:
            raise ValueError(f"codes chunk must be (rows, {self.m_count}), got {codes.shape}")
        if self.rows + codes.shape[0] > self.n:
            raise ValueError(f"{self.path}: more than the declared {self.n} rows")
        self._f.write(np.ascontiguousarray(codes, dtype=f"<u{self.width}").tobytes())
        self.rows += codes.shape[0]

    def close(self) -> None:
        if self._f is None:
            return
        self._f.close()
        self._f = None
        if self.rows != self.n:
            raise ValueError(f"{self.path}: {self.rows} rows written, header declares {self.n}")

    def abort(self) -> None:
        if self._f is not None:
            self._f.close()
            self._f = None
        os.remove(self.path)

    def codes_map(self) -> np.ndarray:
        """Read-only memory map of the written codes (n, M)."""
        if self.n == 0:
            return np.empty((0, self.m_count), dtype=f"<u{self.width}")
        return np.memmap(self.path, dtype=f"<u{self.width}", mode="r", offset=_ENCODED_HEADER,
                         shape=(self.n, self.m_count))

    def __enter__(self):
        return self

    def __exit__(self, et, ev, tb):
        if et is None:
            self.close()
        else:
            self.abort()


def read_encoded(path, mmap: bool = False) -> EncodedDataset:
    """mmap=True maps the codes read-only instead of reading them (large sets)."""
    if mmap:
        with open(path, "rb") as f:
            magic = f.read(4)
            if magic != ENCODED_MAGIC:
                raise FormatError(f"{path}: bad magic {magic!r}, expected {ENCODED_MAGIC!r}", exit_code=2)
            version, n, M, K, width = struct.unpack("<IQIIB", _read_exact(f, 21, path, "header"))
        if version != FORMAT_VERSION:
            raise FormatError(f"{path}: unsupported format version {version}")
        if width not in (1, 2):
            raise FormatError(f"{path}: invalid code width {width}")
        if os.path.getsize(path) < _ENCODED_HEADER + width * n * M:
            raise FormatError(f"{path}: truncated while reading codes")
        codes = (np.memmap(path, dtype=f"<u{width}", mode="r", offset=_ENCODED_HEADER, shape=(n, M)) if n * M
                 else np.empty((n, M), dtype=f"<u{width}"))
        return EncodedDataset(codes=codes, k_count=K)
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != ENCODED_MAGIC:
            raise FormatError(f"{path}: bad magic {magic!r}, expected {ENCODED_MAGIC!r}", exit_code=2)
        version, n, M, K, width = struct.unpack("<IQIIB", _read_exact(f, 21, path, "header"))
        if version != FORMAT_VERSION:
            raise FormatError(f"{path}: unsupported format version {version}")
        if width not in (1, 2):
            raise FormatError(f"{path}: invalid code width {width}")
        codes = np.frombuffer(_read_exact(f, width * n * M, path, "codes"), dtype=f"<u{width}")
        return EncodedDataset(codes=codes.reshape(n, M).copy(), k_count=K)
