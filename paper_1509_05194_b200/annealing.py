"""Dictionary annealing (heat-up / cool-down / re-encode) with device-resident state.

Drop-in for annq/annealing.py: TrainConfig :40-67, TrainStep/TrainReport
:70-94, heat_up :97-112, cool_down :115-126, da_sweep :140-181,
train_from_scratch :225-245, train_online :248-262, rvq_train :265-280.

The data, codes, codebook and cross-product tables stay in HBM for a whole
training call; host arrays are produced only at the return boundary.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _engine as E
from . import codebook as cb
from .validation import check_vectors

__all__ = [
    "TrainConfig",
    "TrainStep",
    "TrainReport",
    "heat_up",
    "cool_down",
    "da_sweep",
    "train_from_scratch",
    "train_online",
    "rvq_train",
]


@dataclass(frozen=True)
class TrainConfig:
    """Training knobs (defaults as annealing.py:40-67; `seed` is only echoed)."""

    m_count: int = 8
    k_count: int = 256
    beam_width: int = 10
    schedule_stages: int = 10
    sweeps: int = 3
    rel_tol: float = 1e-3
    kmeans_iters: int = 30
    seed: int = 0

    def __post_init__(self):
        if self.m_count < 1 or self.k_count < 1:
            raise ValueError("m_count and k_count must be >= 1")
        if self.beam_width < 1:
            raise ValueError("beam_width must be >= 1")
        if self.rel_tol < 0:
            raise ValueError("rel_tol must be >= 0")

    def echo(self) -> dict:
        return {"m": self.m_count, "k": self.k_count, "beam": self.beam_width,
                "stages": self.schedule_stages, "sweeps": self.sweeps, "rel_tol": self.rel_tol,
                "kmeans_iters": self.kmeans_iters, "seed": self.seed}


@dataclass(frozen=True)
class TrainStep:
    sweep: int
    dictionary: int
    distortion: float
    seconds: float


@dataclass
class TrainReport:
    """Per-step log; the distortion column is non-increasing."""

    steps: list = field(default_factory=list)
    config: TrainConfig | None = None

    def record(self, sweep, dictionary, distortion, seconds):
        self.steps.append(TrainStep(sweep, dictionary, float(distortion), float(seconds)))

    def distortions(self) -> np.ndarray:
        return np.array([s.distortion for s in self.steps])

    def rows(self):
        for s in self.steps:
            yield {"sweep": s.sweep, "dictionary": s.dictionary,
                   "distortion": s.distortion, "seconds": s.seconds}


def _codes_dev(encoded, n) -> torch.Tensor:
    codes = np.ascontiguousarray(np.asarray(encoded.codes).astype(np.int32))
    if codes.shape[0] != n:
        raise ValueError(f"codes cover {codes.shape[0]} vectors, data has {n}")
    return E.to_dev(codes)


def heat_up(data, codebook, encoded, m: int) -> np.ndarray:
    """Intermediate set for dictionary m: data minus every other dictionary (float32)."""
    X = check_vectors(data, name="data")
    if encoded.n != X.shape[0]:
        raise ValueError(f"codes cover {encoded.n} vectors, data has {X.shape[0]}")
    if not 0 <= m < codebook.m_count:
        raise ValueError(f"dictionary index {m} out of range [0, {codebook.m_count})")
    cb._raw_kernel()
    cw, _ = cb._codebook_dev(codebook)
    out = E.heat_up(E.to_dev(X), _codes_dev(encoded, X.shape[0]), cw, m)
    return out.cpu().numpy()


def cool_down(intermediate, codebook, m: int, config: TrainConfig):
    """Refit dictionary m to the intermediate set -> (new dict float32 (K,d), assignment int64)."""
    X = check_vectors(intermediate, name="intermediate")
    cw, _ = cb._codebook_dev(codebook)
    new_dict, labels = E.cool_down(E.to_dev(X), cw[m], config)
    return new_dict.cpu().numpy(), labels.cpu().numpy().astype(np.int64)


def _host_codebook(cw: torch.Tensor, order) -> cb.Codebook:
    book = cb.Codebook(codewords=cw.cpu().numpy(), order=np.asarray(order, dtype=np.int64).copy())
    book.__dict__["_dev_cache"] = (book.codewords, cw.device, cw.clone(), E.einsum_sq(cw))
    return book


def da_sweep(data, codebook, encoded, config: TrainConfig, cross=None, sweep_index: int = 1,
             report: TrainReport | None = None):
    """One pass over the M dictionaries -> (codebook, encoded, cross); inputs untouched."""
    X = check_vectors(data, name="data")
    Xd = E.to_dev(X)
    cw0, _ = cb._codebook_dev(codebook)
    cw = cw0.clone()
    if cross is None:
        Pt, sq = E.cross_full(cw)
    else:
        P0, sq0 = cb._cross_dev(cross)
        Pt, sq = P0.clone(), sq0.clone()
    codes = _codes_dev(encoded, X.shape[0])
    E.da_sweep(Xd, cw, codes, Pt, sq, config, sweep_index=sweep_index, report=report)
    book = _host_codebook(cw, codebook.order)
    out = cb.EncodedDataset(codes.cpu().numpy().astype(book.code_dtype), book.k_count,
                            codebook_hash=book.content_hash())
    return book, out, cb.CrossProductTable._from_device(Pt, sq)


def _train_checks(X, config):
    if X.shape[0] < config.k_count:
        raise ValueError(f"need at least k_count={config.k_count} vectors, got {X.shape[0]}")


def train_from_scratch(data, config: TrainConfig):
    """Growth pass from all-zero dictionaries, then up to config.sweeps annealing passes;
    returns a variance-ordered (codebook, encoded, report).  Deterministic."""
    X = check_vectors(data, name="data")
    _train_checks(X, config)
    report = TrainReport(config=config)
    Xd = E.to_dev(X)
    cw, codes = E.growth_pass(Xd, config, report)
    E.sweep_until_converged(Xd, cw, codes, config, report)
    book = cb.Codebook(codewords=cw.cpu().numpy(), order=np.arange(config.m_count, dtype=np.int64))
    book, perm = cb.reorder_by_variance(book)
    codes_h = codes.cpu().numpy()[:, perm]
    encoded = cb.EncodedDataset(codes_h.astype(book.code_dtype), book.k_count, codebook_hash=book.content_hash())
    return book, encoded, report


def train_online(codebook, batch, config: TrainConfig):
    """Encode the batch with the current codebook, then anneal on it (no reorder)."""
    X = check_vectors(batch, name="batch")
    if X.shape[1] != codebook.dim:
        raise ValueError(f"batch d={X.shape[1]} does not match codebook dim {codebook.dim}")
    report = TrainReport(config=config)
    Xd = E.to_dev(X)
    cw0, sq0 = cb._codebook_dev(codebook)
    cw = cw0.clone()
    Pt, sq = E.cross_full(cw)
    codes, _ = E.encode(Xd, cw, sq, Pt, config.beam_width, out_dtype=torch.int32, with_err=False)
    E.sweep_until_converged(Xd, cw, codes, config, report)
    return _host_codebook(cw, codebook.order), report


def rvq_train(data, config: TrainConfig):
    """Greedy residual quantization baseline: the growth pass alone."""
    X = check_vectors(data, name="data")
    _train_checks(X, config)
    Xd = E.to_dev(X)
    cw, codes = E.growth_pass(Xd, config, None)
    book = cb.Codebook(codewords=cw.cpu().numpy(), order=np.arange(config.m_count, dtype=np.int64))
    encoded = cb.EncodedDataset(codes.cpu().numpy().astype(book.code_dtype), book.k_count,
                                codebook_hash=book.content_hash())
    return book, encoded
