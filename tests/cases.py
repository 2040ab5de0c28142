"""Seeded inputs shared by the golden-fixture generator (oracle/make_golden.py)
and the tests.  Everything is regenerated from seeds, so fixtures only store
outputs.  Shapes follow the edge cases the reference suite exercises: tiny d,
K not a multiple of the tile, empty clusters, singletons, n < d (Gram PCA),
beam widths from 1 to full."""

from __future__ import annotations

import numpy as np

BEAM_WIDTHS = (1, 3, 8, 64)
B_TRAIN, B_ENC = 4096, 4096
C_TRAIN, C_ENC = 1536, 512


def mixture(n, d, clusters, spread, seed):
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, 1.0, size=(clusters, d))
    lab = rng.integers(0, clusters, n)
    return (centres[lab] + spread * rng.standard_normal((n, d))).astype(np.float32)


def np_order_inputs():
    rng = np.random.default_rng(1234)
    lengths = [1, 2, 5, 7, 8, 9, 15, 16, 17, 63, 64, 127, 128, 129, 130, 135, 136, 200, 255, 256, 257, 1000,
               1001, 4099, 65537]
    vectors = [rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3, n) for n in lengths]
    dims = [1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 128, 129, 960]
    matrices = [(rng.standard_normal((3, d)) * 10.0 ** rng.uniform(-2, 2, (3, d))).astype(np.float32)
                .astype(np.float64) for d in dims]
    seg_lengths = [1, 2, 3, 7, 8, 9, 10, 17, 64, 65, 128, 129, 130, 131, 137, 300, 1000, 4099]
    seg_arrays = [rng.standard_normal((n, 3)) * 10.0 ** rng.uniform(-3, 3, (n, 3)) for n in seg_lengths]
    return {"vectors": vectors, "matrices": matrices, "seg_arrays": seg_arrays, "seg_lengths": seg_lengths,
            "dims": dims}


def assign_case():
    rng = np.random.default_rng(7)
    X = rng.standard_normal((300, 7))
    C = rng.standard_normal((13, 7))
    C[5] = C[2]  # duplicate centroid: ties must go to the lower index
    return {"X": X, "C": C, "active": 4}


def group_case():
    rng = np.random.default_rng(8)
    k = 37
    labels = rng.integers(0, 30, 2000)  # labels 30..36 stay empty
    labels[:3] = 31  # ...except one small cluster
    labels[5] = 33   # and a singleton
    labels[labels == 2] = 3  # empty label inside the range
    X = rng.standard_normal((2000, 6)) * 10.0 ** rng.uniform(-2, 2, (2000, 6))
    return {"X": X, "labels": labels.astype(np.int64), "k": k}


def lloyd_case():
    X = mixture(400, 5, 8, 0.08, 9).astype(np.float64)
    rng = np.random.default_rng(9)
    C = X[rng.choice(400, 6, replace=False)].copy()
    return {"X": X, "C": C, "active": 3, "iters": 20}


def reseed_case():
    rng = np.random.default_rng(10)
    X = rng.standard_normal((100, 2))
    C = np.vstack([X[:3], [[1e6, 1e6]], [[-1e6, 5.0]]])
    return {"X": X, "C": C, "iters": 10}


def pca_case():
    rng = np.random.default_rng(11)
    X = (rng.standard_normal((200, 6)) * np.array([3.0, 2.0, 1.0, 0.5, 0.1, 0.05])).astype(np.float32)
    Xg = rng.standard_normal((4, 9)).astype(np.float32)
    return {"X": X, "Xgram": Xg}


def staged_case():
    X = mixture(600, 12, 14, 0.06, 12)
    return {"X": X, "C": np.zeros((10, 12)), "iters": 30}


def codebook_case():
    rng = np.random.default_rng(13)
    cw = rng.standard_normal((3, 8, 6)).astype(np.float32)
    cw2 = cw.copy()
    cw2[1] = rng.standard_normal((8, 6)).astype(np.float32)
    X = rng.standard_normal((200, 6)).astype(np.float32)
    q = rng.standard_normal(6)
    return {"cw": cw, "cw2": cw2, "X": X, "q": q}


def sweep_case():
    rng = np.random.default_rng(14)
    X = mixture(400, 8, 10, 0.1, 14)
    cw = rng.standard_normal((3, 8, 8)).astype(np.float32)
    return {"X": X, "cw": cw}


def train_case():
    X = mixture(3000, 16, 30, 0.1, 5)
    X2 = mixture(1500, 16, 30, 0.1, 6)
    return {"X": X, "X2": X2, "config": dict(m_count=4, k_count=16, sweeps=2, beam_width=10, seed=5)}
