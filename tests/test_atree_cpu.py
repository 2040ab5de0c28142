"""A-Tree on the host: the oracle build (oracle/atree_build.py) reproduces the reference's tree arrays, and the
oracle's traversal restatement reproduces the reference's search results
(tests/golden/atree.npz, made by oracle/make_golden_atree.py)."""

import types

import numpy as np
import pytest

import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import atree as AT
from oracle import da_oracle as O
from oracle.atree_build import build_atree_host


@pytest.fixture(scope="module")
def gold():
    import conftest

    return conftest.load_golden("atree.npz")


def _case(g, pre):
    book = da.Codebook(codewords=g[f"{pre}_codewords"], order=g[f"{pre}_order"])
    enc = da.EncodedDataset(codes=g[f"{pre}_codes"], k_count=book.k_count)
    Pm, _ = O.cross_table(book.codewords)
    return book, enc, types.SimpleNamespace(products=Pm)


@pytest.mark.parametrize("pre", ["small", "ties"])
def test_build_matches_reference_tree(gold, pre):
    book, enc, cross = _case(gold, pre)
    t = build_atree_host(enc, book, cross)
    assert t.n_root_children == gold[f"{pre}_tree_meta"][0]
    for f in AT._TREE_FIELDS:
        np.testing.assert_array_equal(getattr(t, f), gold[f"{pre}_tree_{f}"], err_msg=f)
        assert getattr(t, f).dtype == gold[f"{pre}_tree_{f}"].dtype, f


@pytest.mark.parametrize("pre", ["small", "ties"])
def test_oracle_traversal_matches_reference(gold, pre):
    book, enc, cross = _case(gold, pre)
    t = build_atree_host(enc, book, cross)
    Q = gold[f"{pre}_queries"]
    M = book.m_count
    pi = 0
    while f"{pre}_p{pi}_ids" in gold:
        budgets, r = gold[f"{pre}_p{pi}_budgets"], int(gold[f"{pre}_p{pi}_r"][0])
        for qi, q in enumerate(Q):
            vals, qq = O.adc_lut(book.codewords, q)
            ids, d, vis, look, per = O.atree_traverse(vals - qq, qq, t, budgets, r)
            k = len(ids)
            np.testing.assert_array_equal(ids, gold[f"{pre}_p{pi}_ids"][qi, :k])
            assert (gold[f"{pre}_p{pi}_ids"][qi, k:] == -1).all()
            np.testing.assert_array_equal(d, gold[f"{pre}_p{pi}_dists"][qi, :k])
            st = gold[f"{pre}_p{pi}_stats"][qi]
            assert vis == st[0] and look == st[1]
            assert per == [int(v) for v in st[2:2 + M] if v >= 0]
        pi += 1


def test_search_params_budgets():
    np.testing.assert_array_equal(AT.SearchParams(l0=2, ls=2.0, r=5).layer_budgets(4), [4, 8, 16, 32])
    with pytest.raises(ValueError):
        AT.SearchParams(r=0)
    with pytest.raises(ValueError):
        AT.SearchParams(budgets=(1, 2)).layer_budgets(3)
