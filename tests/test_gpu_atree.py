"""GPU A-Tree search against the reference's results (tests/golden/atree.npz).

With the reference's own ADC tables (numpy, via the oracle) uploaded, the GPU
traversal must return the reference's ids, distances and statistics bit for bit.
Through the public API the tables come from the device LUT kernel (float64
within 1e-12 of numpy's dgemv), so ids and statistics are exact and distances
agree to 1e-12 relative."""

import types

import numpy as np
import pytest
import torch

import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E
from paper_1509_05194_b200 import atree as AT
from oracle import da_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    import conftest

    return conftest.load_golden("atree.npz")


def _case(g, pre):
    book = da.Codebook(codewords=g[f"{pre}_codewords"], order=g[f"{pre}_order"])
    enc = da.EncodedDataset(codes=g[f"{pre}_codes"], k_count=book.k_count)
    Pm, _ = O.cross_table(book.codewords)
    tree = AT.build_atree(enc, book, types.SimpleNamespace(products=Pm))
    return book, enc, tree


def _params(g, pre):
    pi = 0
    while f"{pre}_p{pi}_ids" in g:
        yield pi, g[f"{pre}_p{pi}_budgets"], int(g[f"{pre}_p{pi}_r"][0])
        pi += 1


@pytest.mark.parametrize("pre", ["small", "ties"])
def test_traversal_bit_exact_on_reference_tables(gold, pre):
    book, _, tree = _case(gold, pre)
    Q = gold[f"{pre}_queries"]
    tabs = [O.adc_lut(book.codewords, q) for q in Q]
    lut = torch.tensor(np.stack([t[0] for t in tabs]), dtype=torch.float64, device="cuda")
    qsq = torch.tensor([t[1] for t in tabs], dtype=torch.float64, device="cuda")
    M = book.m_count
    for pi, budgets, r in _params(gold, pre):
        ids, d, cnt, st = AT._search_tables(tree, lut, qsq, budgets, r)
        for qi in range(len(Q)):
            k = int(cnt[qi])
            np.testing.assert_array_equal(ids[qi, :k], gold[f"{pre}_p{pi}_ids"][qi, :k])
            assert (gold[f"{pre}_p{pi}_ids"][qi, k:] == -1).all()
            np.testing.assert_array_equal(d[qi, :k], gold[f"{pre}_p{pi}_dists"][qi, :k])
            np.testing.assert_array_equal(st[qi], gold[f"{pre}_p{pi}_stats"][qi])


@pytest.mark.parametrize("pre", ["small", "ties"])
def test_public_search_matches_reference(gold, pre):
    book, _, tree = _case(gold, pre)
    Q = gold[f"{pre}_queries"]
    for pi, budgets, r in _params(gold, pre):
        params = AT.SearchParams(r=r, budgets=tuple(int(b) for b in budgets))
        ids, d, cnt, st = AT.atree_search_batch(tree, book, Q, params)
        for qi in range(len(Q)):
            k = int(cnt[qi])
            np.testing.assert_array_equal(ids[qi, :k], gold[f"{pre}_p{pi}_ids"][qi, :k])
            np.testing.assert_allclose(d[qi, :k], gold[f"{pre}_p{pi}_dists"][qi, :k], rtol=1e-12, atol=1e-12)
            np.testing.assert_array_equal(st[qi], gold[f"{pre}_p{pi}_stats"][qi])
        one_ids, one_d, stats = AT.atree_search(tree, book, Q[0], params)
        np.testing.assert_array_equal(one_ids, ids[0, :int(cnt[0])])
        assert stats.nodes_visited == st[0, 0]


def test_unbounded_budgets_match_exhaustive_adc(gold):
    book, enc, tree = _case(gold, "small")
    Q = gold["small_queries"][:6]
    n = enc.n
    params = AT.SearchParams(r=20, budgets=(n,) * book.m_count)
    ids, d, cnt, _ = AT.atree_search_batch(tree, book, Q, params)
    eids, ed = da.exhaustive_adc_search_batch(book, enc, Q, 20)
    np.testing.assert_array_equal(ids, eids)
    # tree distances carry float32 epsilons (atree.py:150-155): the reference allows 1e-3
    np.testing.assert_allclose(d, ed, rtol=1e-3, atol=1e-8)


def test_brute_force_knn_matches_reference():
    import conftest
    from paper_1509_05194_b200.groundtruth import brute_force_knn

    g = conftest.load_golden("knn.npz")
    for r in (1, 10, 37):
        gt = brute_force_knn(g["base"], g["queries"], r)
        np.testing.assert_array_equal(gt.ids, g[f"r{r}_ids"])
        np.testing.assert_array_equal(gt.distances, g[f"r{r}_dists"])
    with pytest.raises(ValueError):
        brute_force_knn(g["base"], g["queries"][:, :3], 5)
