"""Behavioural properties the reference's own suite checks (pkg/tests/test_codebook.py,
test_atree.py), restated against this implementation on the GPU: single-dictionary
encode is nearest-codeword, a full beam is exhaustive, ADC identities, the A-Tree's
structural invariants, accounting and edge cases."""

import itertools
import types

import numpy as np
import pytest

import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import atree as AT
from oracle import da_oracle as O

pytestmark = pytest.mark.gpu


def book_of(rng, M, K, D):
    return da.Codebook(codewords=rng.standard_normal((M, K, D)).astype(np.float32), order=np.arange(M))


def test_single_dictionary_encode_is_nearest_codeword():
    rng = np.random.default_rng(1)
    book = book_of(rng, 1, 32, 9)
    X = rng.standard_normal((500, 9)).astype(np.float32)
    codes = da.encode_dataset(book, X, beam_width=4).codes[:, 0].astype(np.int64)
    c64 = book.codewords[0].astype(np.float64)
    d2 = ((X.astype(np.float64)[:, None, :] - c64[None]) ** 2).sum(-1)
    best = d2.min(axis=1)
    # the chosen codeword attains the minimum (up to the reference's expanded-form rounding)
    np.testing.assert_allclose(d2[np.arange(500), codes], best, rtol=1e-9, atol=1e-9)


def test_full_beam_is_exhaustive():
    rng = np.random.default_rng(2)
    M, K, D = 3, 4, 5
    book = book_of(rng, M, K, D)
    X = rng.standard_normal((200, D)).astype(np.float32)
    enc = da.encode_dataset(book, X, beam_width=K ** (M - 1))
    err = da.distortion(book, X, enc) if hasattr(da, "distortion") else None
    c64 = book.codewords.astype(np.float64)
    allc = np.array(list(itertools.product(range(K), repeat=M)))
    rec = sum(c64[m][allc[:, m]] for m in range(M))
    d2 = ((X.astype(np.float64)[:, None, :] - rec[None]) ** 2).sum(-1)
    got = sum(c64[m][enc.codes[:, m].astype(np.int64)] for m in range(M))
    mine = ((X.astype(np.float64) - got) ** 2).sum(-1)
    np.testing.assert_allclose(mine, d2.min(axis=1), rtol=1e-9, atol=1e-9)
    assert err is None or np.isfinite(err)


def test_encode_is_deterministic():
    rng = np.random.default_rng(3)
    book = book_of(rng, 4, 16, 12)
    X = rng.standard_normal((3000, 12)).astype(np.float32)
    a = da.encode_dataset(book, X, beam_width=6).codes
    b = da.encode_dataset(book, X, beam_width=6).codes
    np.testing.assert_array_equal(a, b)


def test_adc_table_identities():
    rng = np.random.default_rng(4)
    book = book_of(rng, 3, 8, 6)
    # query equal to one codeword: that entry is 0
    q = book.codewords[1, 5].astype(np.float64)
    t = da.adc_table(book, q)
    assert t.values[1, 5] == pytest.approx(0.0, abs=1e-12)
    # zero query: entries are the codeword norms, ||q||^2 = 0
    t0 = da.adc_table(book, np.zeros(6))
    np.testing.assert_allclose(t0.values, (book.codewords.astype(np.float64) ** 2).sum(-1), rtol=1e-12)
    assert t0.q_sq_norm == 0.0


def test_adc_exact_match_ranks_first_and_pair_sums_consistent():
    rng = np.random.default_rng(5)
    M, K, D = 3, 8, 6
    book = book_of(rng, M, K, D)
    codes = rng.integers(0, K, size=(400, M)).astype(np.uint8)
    codes = np.unique(codes, axis=0)
    enc = da.EncodedDataset(codes=codes, k_count=K)
    cross = da.cross_products(book)
    i = 17
    q = sum(book.codewords[m, codes[i, m]].astype(np.float64) for m in range(M))
    ids, d = da.exhaustive_adc_search(book, enc, q, 3, cross=cross)
    assert ids[0] == i and d[0] == pytest.approx(0.0, abs=1e-9)
    with pytest.raises(ValueError):
        da.exhaustive_adc_search(book, enc, q, enc.n + 1, cross=cross)
    pair = da.code_pair_sums(cross, codes)
    t = da.adc_table(book, q)
    for j in (0, 5, 40):
        direct = da.adc_distance(t, cross, codes[j])
        via = sum(t.values[m, codes[j, m]] for m in range(M)) - (M - 1) * t.q_sq_norm + pair[j]
        assert via == pytest.approx(direct, rel=1e-12, abs=1e-12)


def _tree(book, codes, K):
    enc = da.EncodedDataset(codes=np.asarray(codes), k_count=K)
    Pm, _ = O.cross_table(book.codewords)
    return enc, AT.build_atree(enc, book, types.SimpleNamespace(products=Pm))


def test_atree_structure_and_edge_cases():
    rng = np.random.default_rng(6)
    book = book_of(rng, 3, 4, 6)
    # one vector: a single leaf hanging off the root
    _, t1 = _tree(book, np.array([[1, 2, 3]], dtype=np.uint8), 4)
    assert t1.n_root_children == 1 and t1.leaf_count == 1 and t1.internal_count == 0
    for l0 in (1, 7):
        ids, _, _ = AT.atree_search(t1, book, np.zeros(6), AT.SearchParams(l0=l0, ls=1.0, r=3))
        np.testing.assert_array_equal(ids, [0])
    # duplicate codes collapse into one leaf carrying every id
    codes = np.array([[1, 2, 3], [1, 2, 3], [1, 2, 0], [1, 2, 3]], dtype=np.uint8)
    enc, t2 = _tree(book, codes, 4)
    assert t2.leaf_count == 2
    np.testing.assert_array_equal(np.sort(t2.leaf_ids), np.arange(4))
    # r beyond the survivors: every id of every surviving leaf (here one leaf per layer budget)
    ids, d, st = AT.atree_search(t2, book, np.zeros(6), AT.SearchParams(l0=1, ls=1.0, r=50))
    v, qq = O.adc_lut(book.codewords, np.zeros(6))
    o_ids, _, _, _, _ = O.atree_traverse(v - qq, qq, t2, np.ones(3, dtype=np.int64), 50)
    np.testing.assert_array_equal(ids, o_ids)
    assert 0 < ids.size < 50
    ids, d, st = AT.atree_search(t2, book, np.zeros(6), AT.SearchParams(budgets=(9, 9, 9), r=50))
    assert sorted(ids.tolist()) == [0, 1, 2, 3]          # budgets wide enough: everything
    assert st.nodes_visited <= t2.node_count
    assert st.table_lookups >= st.nodes_visited
    # zero query: distance = squared norm of the reconstruction
    recs = {tuple(c): sum(book.codewords[m, c[m]].astype(np.float64) for m in range(3)) for c in codes.tolist()}
    for i, di in zip(ids, d):
        assert di == pytest.approx(float((recs[tuple(codes[i].tolist())] ** 2).sum()), rel=1e-5, abs=1e-6)
    # empty dataset and wrong codebook
    _, t0 = _tree(book, np.zeros((0, 3), dtype=np.uint8), 4)
    ids, d, _ = AT.atree_search(t0, book, np.zeros(6), AT.SearchParams(r=5))
    assert ids.size == 0 and d.size == 0
    other = book_of(np.random.default_rng(7), 3, 4, 6)
    with pytest.raises(da.FormatError):
        AT.atree_search(t2, other, np.zeros(6), AT.SearchParams(r=1))


def test_atree_recall_monotone_in_budget():
    rng = np.random.default_rng(8)
    M, K, D = 4, 16, 16
    book = book_of(rng, M, K, D)
    X = rng.standard_normal((4000, D)).astype(np.float32)
    enc = da.encode_dataset(book, X, beam_width=4)
    _, tree = _tree(book, enc.codes, K)
    Q = rng.standard_normal((60, D))
    eids, _ = da.exhaustive_adc_search_batch(book, enc, Q, 10)
    recalls, visited = [], []
    for l0 in (1, 2, 4, 8, 16, 64):
        ids, _, _, st = AT.atree_search_batch(tree, book, Q, AT.SearchParams(l0=l0, ls=2.0, r=10))
        recalls.append(np.mean([len(set(a) & set(b)) for a, b in zip(ids, eids)]) / 10)
        visited.append(st[:, 0].mean())
    assert all(b >= a - 1e-12 for a, b in zip(recalls, recalls[1:])), recalls
    assert all(b >= a for a, b in zip(visited, visited[1:])), visited
    assert recalls[-1] > 0.9
