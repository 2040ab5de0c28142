"""Exact k-NN ground truth on the GPU (data.py:167-215).

`brute_force_knn(base, queries, r)`: squared L2 in float64 with the reference's
expansion `max((||q||^2 - 2 q.x) + ||x||^2, 0)`, the dot product in OpenBLAS
dgemm order and the row norms as numpy pairwise sums, top-r per query with ties
to the lower id.  Distance blocks are formed by the ordered GEMM kernel and
reduced by a per-row radix-select kernel (`da_knn`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _engine as E
from ._engine import P
from ._native import native
from .validation import check_vectors

__all__ = ["GroundTruth", "brute_force_knn"]


@dataclass(frozen=True)
class GroundTruth:
    """Exact top-r neighbours per query (data.py:31-45)."""

    ids: np.ndarray
    distances: np.ndarray

    @property
    def n_queries(self) -> int:
        return self.ids.shape[0]

    @property
    def r(self) -> int:
        return self.ids.shape[1]


def brute_force_knn(base, queries, r: int, n_jobs: int = 1) -> GroundTruth:
    """Exact squared-L2 top-r per query; ties broken by lower id.  n_jobs is accepted
    for API compatibility (the device computes every block)."""
    base = check_vectors(base, name="base")
    queries = check_vectors(queries, name="queries")
    if base.shape[1] != queries.shape[1]:
        raise ValueError(f"dimension mismatch: base d={base.shape[1]}, queries d={queries.shape[1]}")
    if r < 1 or r > base.shape[0]:
        raise ValueError(f"r={r} must be in [1, {base.shape[0]}]")
    n, D = base.shape
    nq = queries.shape[0]
    B = E.to_dev(base)                                   # float32 rows, widened exactly in the GEMM
    Q = E.to_dev(queries).to(torch.float64)
    bsq = E.row_sqnorms(B, D)
    qsq = E.row_sqnorms(Q, D)
    ids = torch.empty((nq, r), dtype=torch.int64, device=B.device)
    d = torch.empty((nq, r), dtype=torch.float64, device=B.device)
    if nq:
        native.da_knn(P(B), 1, n, B.stride(0), D, P(bsq), P(Q), nq, P(qsq), int(r), P(ids), P(d), E.stream())
    return GroundTruth(ids=ids.cpu().numpy(), distances=d.cpu().numpy())
