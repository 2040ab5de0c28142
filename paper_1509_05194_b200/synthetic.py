"""Frozen seeded generators for the BASELINE.json configurations.

The public datasets the paper uses (SIFT1M, GIST1M, SIFT1B) are not
available; these mixtures stand in for them with the stated shapes, ranges
and value distributions.  Draw order is fixed: component means, then labels,
then noise, so every run (oracle, GPU, any machine) sees identical bytes.
Large sets are generated chunk by chunk from named substreams.
"""

from __future__ import annotations

import numpy as np

from .validation import substream

__all__ = ["config_a", "config_b", "config_c", "mixture_b_params", "mixture_b_chunk", "config_e_queries",
           "config_e_candidates"]


def config_a(n=10_000, d=32, comps=64, sigma=0.3, seed=0) -> np.ndarray:
    """CPU-runnable DA: 64-component isotropic mixture, centres ~ N(0, I), sigma 0.3."""
    rng = np.random.default_rng(seed)
    centres = rng.standard_normal((comps, d))
    labels = rng.integers(0, comps, n)
    x = centres[labels] + sigma * rng.standard_normal((n, d))
    return x.astype(np.float32)


def mixture_b_params(seed=1, comps=1024, d=128) -> np.ndarray:
    """Per-component means ~ U[0, 60]^d (config B / D / E mixture)."""
    return np.random.default_rng(seed).uniform(0.0, 60.0, size=(comps, d))


def _draw_b(rng, means, n, sigma=20.0) -> np.ndarray:
    labels = rng.integers(0, means.shape[0], n)
    x = np.abs(means[labels] + sigma * rng.standard_normal((n, means.shape[1])))
    return np.clip(np.rint(x), 0, 255)


def config_b(n=1_000_000, seed=1, chunk=250_000) -> np.ndarray:
    """Integer-valued float32 in [0, 255], D=128 (SIFT-like), heavy right tail via |x|."""
    means = mixture_b_params(seed)
    out = np.empty((n, means.shape[1]), dtype=np.float32)
    for c0 in range(0, n, chunk):
        rng = substream(seed, f"b-chunk-{c0 // chunk}")
        out[c0:c0 + chunk] = _draw_b(rng, means, min(chunk, n - c0))
    return out


def mixture_b_chunk(seed: int, chunk_index: int, n=1_000_000, params_seed=1) -> np.ndarray:
    """Config D/E stream chunk: config-B mixture (means from params_seed), stored uint8."""
    means = mixture_b_params(params_seed)
    rng = substream(seed, f"chunk-{chunk_index}")
    return _draw_b(rng, means, n).astype(np.uint8)


def config_c(n=1_000_000, d=960, comps=512, seed=2, chunk=100_000) -> np.ndarray:
    """High-dim: means ~ U[0, 0.3]^960, sigma 0.05, clipped to [0, 1] (GIST-like)."""
    means = np.random.default_rng(seed).uniform(0.0, 0.3, size=(comps, d))
    out = np.empty((n, d), dtype=np.float32)
    for c0 in range(0, n, chunk):
        rng = substream(seed, f"c-chunk-{c0 // chunk}")
        m = min(chunk, n - c0)
        lab = rng.integers(0, comps, m)
        out[c0:c0 + m] = np.clip(means[lab] + 0.05 * rng.standard_normal((m, d)), 0.0, 1.0)
    return out


def config_e_queries(nq=10_000, seed=4) -> np.ndarray:
    means = mixture_b_params(1)
    rng = substream(seed, "queries")
    lab = rng.integers(0, means.shape[0], nq)
    return np.abs(means[lab] + 20.0 * rng.standard_normal((nq, means.shape[1]))).astype(np.float32)


def config_e_candidates(nq: int, ncand=100_000, n_total=1_000_000_000, seed=4) -> np.ndarray:
    """Per query `ncand` distinct uniform ids in [0, n_total), sorted ascending."""
    rng = substream(seed, "candidates")
    out = np.empty((nq, ncand), dtype=np.int64)
    for i in range(nq):
        ids = np.unique(rng.integers(0, n_total, int(ncand * 1.01) + 16))
        while ids.size < ncand:
            ids = np.unique(np.concatenate([ids, rng.integers(0, n_total, ncand)]))
        out[i] = np.sort(rng.choice(ids, ncand, replace=False))
    return out
