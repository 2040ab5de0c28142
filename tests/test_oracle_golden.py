"""Pin the CPU oracle against outputs of the REFERENCE itself (tests/golden,
made by oracle/make_golden.py).  The oracle is the checker for every GPU
parity test, so it must reproduce the reference bit-for-bit here."""

import numpy as np
import pytest

import cases
from oracle import da_oracle as O


def test_assign(golden):
    g, c = golden("small_ops.npz"), cases.assign_case()
    lab, d2 = O.nearest(c["X"][:, : c["active"]], c["C"][:, : c["active"]])
    np.testing.assert_array_equal(lab, g["assign_labels"])
    np.testing.assert_array_equal(d2, g["assign_d2"])


def test_group_means(golden):
    g, c = golden("small_ops.npz"), cases.group_case()
    means, counts = O.segment_means(c["X"], c["labels"], c["k"])
    np.testing.assert_array_equal(means, g["group_means"])
    np.testing.assert_array_equal(counts, g["group_counts"])


@pytest.mark.parametrize("which", ["lloyd", "reseed"])
def test_lloyd(golden, which):
    g = golden("small_ops.npz")
    c = cases.lloyd_case() if which == "lloyd" else cases.reseed_case()
    C, lab, tr = O.lloyd(c["X"], c["C"], c.get("active", c["X"].shape[1]), c["iters"])
    np.testing.assert_array_equal(C, g[f"{which}_points"])
    np.testing.assert_array_equal(lab, g[f"{which}_assign"])
    np.testing.assert_array_equal(np.array(tr), g[f"{which}_trace"])


def test_pca(golden):
    g, c = golden("small_ops.npz"), cases.pca_case()
    R, mu = O.pca(c["X"].astype(np.float64))
    np.testing.assert_array_equal(R, g["pca_rotation"])
    np.testing.assert_array_equal(mu, g["pca_mean"])
    Rg, mug = O.pca(c["Xgram"].astype(np.float64))
    np.testing.assert_array_equal(Rg, g["pcag_rotation"])


def test_staged_kmeans(golden):
    g, c = golden("small_ops.npz"), cases.staged_case()
    pts, lab, tr = O.staged_kmeans(c["X"].astype(np.float64), c["C"], O.schedule(c["X"].shape[1]), c["iters"])
    np.testing.assert_array_equal(pts, g["staged_points"])
    np.testing.assert_array_equal(lab, g["staged_assign"])
    np.testing.assert_array_equal(np.array(tr), g["staged_trace"])


def test_cross_and_refresh(golden):
    g, c = golden("small_ops.npz"), cases.codebook_case()
    P, sq = O.cross_table(c["cw"])
    np.testing.assert_array_equal(P, g["cross_P"])
    np.testing.assert_array_equal(sq, g["cross_sq"])
    P2, sq2 = O.cross_refresh(P, sq, c["cw2"], 1)
    np.testing.assert_array_equal(P2, g["refresh_P"])
    np.testing.assert_array_equal(sq2, g["refresh_sq"])


@pytest.mark.parametrize("L", cases.BEAM_WIDTHS)
def test_beam(golden, L):
    g, c = golden("small_ops.npz"), cases.codebook_case()
    P, _ = O.cross_table(c["cw"])
    codes, errs = O.beam_encode(c["cw"].astype(np.float64), P, c["X"].astype(np.float64), L)
    np.testing.assert_array_equal(codes, g[f"beam_codes_L{L}"])
    np.testing.assert_array_equal(errs, g[f"beam_errs_L{L}"])
    np.testing.assert_array_equal(O.encode_chunked(c["cw"], P, c["X"], L), g[f"enc_codes_L{L}"])


def test_adc(golden):
    g, c = golden("small_ops.npz"), cases.codebook_case()
    v, qq = O.adc_lut(c["cw"], c["q"])
    np.testing.assert_array_equal(v, g["adc_values"])
    assert qq == float(g["adc_qsq"])
    P, _ = O.cross_table(c["cw"])
    codes = O.encode_chunked(c["cw"], P, c["X"], 8)
    pair = O.pair_terms(P, codes)
    np.testing.assert_array_equal(pair, g["pair_sums"])
    pos, d = O.adc_topr(v, qq, codes, pair, 10)
    np.testing.assert_array_equal(pos, g["search_ids"])
    np.testing.assert_array_equal(d, g["search_dists"])


def test_heat_cool_sweep(golden):
    g, c = golden("small_training.npz"), cases.sweep_case()
    P, sq = O.cross_table(c["cw"])
    codes = O.encode_chunked(c["cw"], P, c["X"], 8)
    np.testing.assert_array_equal(codes, g["sweep_init_codes"])
    inter = O.heat_up(c["X"], c["cw"], codes, 1)
    np.testing.assert_array_equal(inter, g["heat_up_1"])
    nd, lab = O.cool_down(inter, c["cw"], 1, 10, 30)
    np.testing.assert_array_equal(nd, g["cool_dict"])
    np.testing.assert_array_equal(lab, g["cool_assign"])
    steps = []
    cw2, codes2, P2, _ = O.sweep(c["X"], c["cw"], codes, P, sq, 8, 10, 30, steps)
    np.testing.assert_array_equal(cw2, g["sweep_cw"])
    np.testing.assert_array_equal(codes2, g["sweep_codes"])
    np.testing.assert_array_equal(np.array([s[2] for s in steps]), g["sweep_dist"])
    np.testing.assert_array_equal(P2, g["sweep_P"])


def test_train_small(golden):
    g, c = golden("small_training.npz"), cases.train_case()
    k = c["config"]
    cw, codes, steps, perm = O.train_from_scratch(c["X"], k["m_count"], k["k_count"], L=k["beam_width"],
                                                  sweeps=k["sweeps"])
    np.testing.assert_array_equal(cw, g["train_cw"])
    np.testing.assert_array_equal(perm, g["train_order"])
    np.testing.assert_array_equal(codes, g["train_codes"])
    np.testing.assert_array_equal(np.array([s[2] for s in steps]), g["train_dist"])
    rcw, rcodes = O.growth(c["X"], k["m_count"], k["k_count"], 10, 30)
    np.testing.assert_array_equal(rcw, g["rvq_cw"])
    np.testing.assert_array_equal(rcodes, g["rvq_codes"])
    ocw, osteps = O.train_online(g["train_cw"], c["X2"], L=k["beam_width"], sweeps=k["sweeps"])
    np.testing.assert_array_equal(ocw, g["online_cw"])
    np.testing.assert_array_equal(np.array([s[2] for s in osteps]), g["online_dist"])
