"""PCA rotation and staged (incremental-dimension) Lloyd k-means on the B200.

Drop-in for annq/clustering.py: PcaModel :31-43, Centroids :46-60,
pca_fit :82-113, dimension_schedule :116-131, lloyd_kmeans :165-203,
quantization_error :206-212, improved_kmeans :215-250.  The Lloyd loop runs
on the device (assign kernel + bit-exact reduceat group means); only the
per-iteration stable/empty tests and LAPACK's eigh touch the host.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _engine as E
from .validation import check_vectors

__all__ = [
    "PcaModel",
    "Centroids",
    "pca_fit",
    "dimension_schedule",
    "lloyd_kmeans",
    "improved_kmeans",
    "quantization_error",
]

dimension_schedule = E.dimension_schedule


@dataclass(frozen=True)
class PcaModel:
    """Orthonormal rotation (rows = components, descending variance) and centre."""

    rotation: np.ndarray
    mean: np.ndarray
    explained_variance: np.ndarray

    def _apply(self, X, inverse: bool) -> np.ndarray:
        A = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
        squeeze = A.ndim == 1
        if squeeze:
            A = A.reshape(1, -1)
        R = E.to_dev(np.ascontiguousarray(self.rotation, dtype=np.float64))
        mu = E.to_dev(np.ascontiguousarray(self.mean, dtype=np.float64))
        out = E.rotate(E.to_dev(A), R, mu, inverse=inverse).cpu().numpy()
        return out[0] if squeeze else out

    def transform(self, X) -> np.ndarray:
        """(X - mean) @ rotation.T"""
        return self._apply(X, inverse=False)

    def inverse_transform(self, Y) -> np.ndarray:
        """Y @ rotation + mean"""
        return self._apply(Y, inverse=True)


@dataclass
class Centroids:
    """k centroids, the nearest-centroid assignment, and the Lloyd objective trace."""

    points: np.ndarray
    assignment: np.ndarray
    objective_trace: list = field(default_factory=list)

    @property
    def k(self) -> int:
        return self.points.shape[0]


def _centroid_points(init) -> np.ndarray:
    pts = init.points if isinstance(init, Centroids) or hasattr(init, "assignment") else init
    return np.asarray(pts, dtype=np.float64)


def pca_fit(data) -> PcaModel:
    """Full orthonormal PCA of the centred data (covariance on the device, eigh in LAPACK)."""
    X = check_vectors(data, dtype=np.float64, name="data")
    n = X.shape[0]
    if n < 2:
        raise ValueError(f"PCA needs at least 2 vectors, got {n}")
    R_d, mean_d, variances, R_h = E.pca(E.to_dev(X))
    return PcaModel(rotation=R_h, mean=mean_d.cpu().numpy(), explained_variance=variances)


def lloyd_kmeans(data, init, active_dims: int | None = None, max_iters: int = 30) -> Centroids:
    """Lloyd iterations on the leading active_dims coordinates (means over all)."""
    X = np.ascontiguousarray(np.asarray(data, dtype=np.float64))
    C = _centroid_points(init).copy()
    n, d = X.shape
    k = C.shape[0]
    if k > n:
        raise ValueError(f"k={k} exceeds the number of points n={n}")
    if active_dims is None:
        active_dims = d
    if not 1 <= active_dims <= d:
        raise ValueError(f"active_dims={active_dims} must be in [1, {d}]")
    Cd, labels, trace = E.lloyd(E.to_dev(X), E.to_dev(np.ascontiguousarray(C)), active_dims, max_iters)
    return Centroids(points=Cd.cpu().numpy(), assignment=labels.cpu().numpy().astype(np.int64),
                     objective_trace=trace)


def quantization_error(data, centroids, active_dims: int | None = None) -> float:
    """Mean squared distance of each point to its nearest centroid."""
    X = np.ascontiguousarray(np.asarray(data, dtype=np.float64))
    C = np.ascontiguousarray(_centroid_points(centroids))
    a = X.shape[1] if active_dims is None else active_dims
    _, errs = E.assign(E.to_dev(X), a, E.to_dev(C))
    return float(E.np_mean(errs).item())


def improved_kmeans(data, init, schedule: list[int] | None = None, max_iters: int = 30) -> Centroids:
    """Staged k-means in PCA space; never worse than init on the full dimension."""
    X = np.ascontiguousarray(np.asarray(data, dtype=np.float64))
    C0 = np.ascontiguousarray(_centroid_points(init))
    d = X.shape[1]
    if schedule is None:
        schedule = dimension_schedule(d)
    if schedule[-1] != d:
        raise ValueError(f"schedule must end at d={d}, got {schedule}")
    E.check_k(X.shape[0], C0.shape[0])
    pts, labels, trace = E.improved_kmeans(E.to_dev(X), E.to_dev(C0), list(schedule), max_iters)
    return Centroids(points=pts.cpu().numpy(), assignment=labels.cpu().numpy().astype(np.int64),
                     objective_trace=trace)
