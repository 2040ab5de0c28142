"""The float64 association orders the CUDA kernels reproduce (csrc/common.cuh),
pinned against numpy itself and against the reference's fixtures."""

import numpy as np

import cases
from oracle import np_order


def test_pairwise_matches_numpy(golden):
    g = golden("np_order.npz")
    c = cases.np_order_inputs()
    for i, v in enumerate(c["vectors"]):
        assert np_order.pairwise(v) == v.sum() == g["pairwise"][i]
        assert np_order.pairwise(v * v) == (v * v).sum() == g["rowsum"][i]
        assert np_order.pairwise(v) / len(v) == v.mean() == g["mean"][i]


def test_reduceat_is_first_plus_pairwise(golden):
    g = golden("np_order.npz")
    c = cases.np_order_inputs()
    got = np.concatenate([[np_order.reduceat_segment(a[:, j]) for j in range(a.shape[1])]
                          for a in c["seg_arrays"]])
    np.testing.assert_array_equal(got, g["reduceat"])


def test_einsum_sq_order(golden):
    g = golden("np_order.npz")
    c = cases.np_order_inputs()
    got = np.concatenate([[np_order.einsum_sq(row) for row in m] for m in c["matrices"]])
    np.testing.assert_array_equal(got, g["einsum"])
    for m in c["matrices"]:
        np.testing.assert_array_equal([np_order.einsum_sq(r) for r in m], np.einsum("kd,kd->k", m, m))


def test_axis0_mean_is_sequential():
    rng = np.random.default_rng(3)
    X = rng.standard_normal((1000, 4)) * 10.0 ** rng.uniform(-3, 3, (1000, 4))
    for j in range(4):
        s = 0.0
        for v in X[:, j]:
            s += v
        assert s / 1000 == X.mean(axis=0)[j]
