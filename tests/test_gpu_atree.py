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


@pytest.mark.parametrize("pre", ["small", "ties"])
def test_device_build_matches_reference_tree(gold, pre):
    """The GPU build (radix passes + device scans) gives the reference's arrays."""
    book = da.Codebook(codewords=gold[f"{pre}_codewords"], order=gold[f"{pre}_order"])
    enc = da.EncodedDataset(codes=gold[f"{pre}_codes"], k_count=book.k_count)
    Pm, _ = O.cross_table(book.codewords)
    t = AT.build_atree(enc, book, types.SimpleNamespace(products=Pm))
    assert t.n_root_children == gold[f"{pre}_tree_meta"][0]
    for f in AT._TREE_FIELDS:
        np.testing.assert_array_equal(getattr(t, f), gold[f"{pre}_tree_{f}"], err_msg=f)
        assert getattr(t, f).dtype == gold[f"{pre}_tree_{f}"].dtype, f


@pytest.mark.parametrize("M,K,n,dup,idmap", [(4, 16, 20000, 0.3, False), (8, 256, 200000, 0.05, True),
                                             (3, 5, 4000, 0.5, True), (1, 8, 100, 0.0, False)])
def test_device_build_matches_host_build(M, K, n, dup, idmap):
    """Device build == the oracle's host restatement on larger, duplicate-heavy
    code sets, with and without an id_map (ids ascending inside each leaf)."""
    from oracle.atree_build import build_atree_host

    rng = np.random.default_rng(M * 1000 + K)
    cw = rng.standard_normal((M, K, 6)).astype(np.float32)
    book = da.Codebook(codewords=cw, order=np.arange(M))
    base = rng.integers(0, K, (max(1, int(n * (1 - dup))), M))
    codes = base[rng.integers(0, len(base), n)].astype(np.uint8 if K <= 256 else np.uint16)
    id_map = rng.permutation(10 * n)[:n].astype(np.int64) if idmap else None
    enc = da.EncodedDataset(codes=codes, k_count=K, id_map=id_map)
    Pm, _ = O.cross_table(cw)
    cross = types.SimpleNamespace(products=Pm)
    a = AT.build_atree(enc, book, cross)
    b = build_atree_host(enc, book, cross)
    assert a.n_root_children == b.n_root_children
    for f in AT._TREE_FIELDS:
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)
        assert getattr(a, f).dtype == getattr(b, f).dtype, f
