"""The filtered encoder (fp32 tables + rigorous bound + exact float64 recheck)
must return exactly what the plain float64 encoder returns: same codes, same
float64 errors, for every beam width, including ties and degenerate books."""

import numpy as np
import pytest
import torch

import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E
from paper_1509_05194_b200 import codebook as cb
from paper_1509_05194_b200 import synthetic

pytestmark = pytest.mark.gpu


def both(book, X, L):
    """(tensor-core filter, plain float64, rechecked count); also checks the fp32
    gather filter against the plain encoder."""
    cross = cb.cross_products(book)
    cw, sq = cb._codebook_dev(book)
    Pt, _ = cross.device()
    Xd = E.to_dev(X)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    E.encode_config(3, cnt)
    tc = E.encode(Xd, cw, sq, Pt, L)
    E.encode_config(2)
    gather = E.encode(Xd, cw, sq, Pt, L)
    E.encode_config(1)
    plain = E.encode(Xd, cw, sq, Pt, L)
    E.encode_config(0)
    assert_same(gather, plain)
    return tc, plain, int(cnt.item())


def assert_same(fast, plain):
    np.testing.assert_array_equal(fast[0].cpu().numpy(), plain[0].cpu().numpy())
    np.testing.assert_array_equal(fast[1].cpu().numpy(), plain[1].cpu().numpy())


@pytest.mark.parametrize("L", [1, 2, 5, 10, 16, 40, 64])
def test_random_books(L):
    rng = np.random.default_rng(L)
    for M, K, D in [(3, 8, 6), (4, 16, 17), (2, 300, 9), (8, 256, 128)]:
        book = da.Codebook(codewords=rng.standard_normal((M, K, D)).astype(np.float32), order=np.arange(M))
        X = rng.standard_normal((700, D)).astype(np.float32)
        fast, plain, _ = both(book, X, L)
        assert_same(fast, plain)


def test_ties_and_zero_book():
    book = da.Codebook.zeros(3, 4, 2)
    X = np.array([[1.0, 2.0], [0.0, 0.0], [-3.0, 1.0]], dtype=np.float32)
    for L in (1, 4, 16):
        fast, plain, _ = both(book, X, L)
        assert_same(fast, plain)
        assert (fast[0].cpu().numpy() == 0).all()
    rng = np.random.default_rng(3)
    cw = rng.standard_normal((3, 6, 5)).astype(np.float32)
    cw[1, 4] = cw[1, 1]          # duplicate codewords -> exact score ties
    cw[2] = cw[2][[0, 0, 2, 2, 4, 4]]
    book = da.Codebook(codewords=cw, order=np.arange(3))
    X = rng.standard_normal((400, 5)).astype(np.float32)
    for L in (1, 3, 7):
        fast, plain, _ = both(book, X, L)
        assert_same(fast, plain)


def test_config_b_like_and_recheck_rate():
    X = synthetic.config_b(n=30_000, chunk=10_000)
    cfg = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
    book, _, _ = da.train_from_scratch(X[:5000], cfg)
    for L in (1, 10):
        fast, plain, rechecked = both(book, X, L)
        assert_same(fast, plain)
        # candidates per vector: sum over stages of live*K; the filter must cut most of them
        total = X.shape[0] * sum(min(L, 256 ** m) * 256 for m in range(1, 9))
        assert rechecked < 0.05 * total, (rechecked, total)


def test_streamed_host_encode_matches_device_encode():
    rng = np.random.default_rng(11)
    book = da.Codebook(codewords=rng.standard_normal((4, 16, 12)).astype(np.float32), order=np.arange(4))
    X = rng.standard_normal((2500, 12)).astype(np.float32)
    cross = cb.cross_products(book)
    cw, sq = cb._codebook_dev(book)
    Pt, _ = cross.device()
    ref, _ = E.encode(E.to_dev(X), cw, sq, Pt, 5, with_err=False)
    for chunk in (1000, 2500, 4096):
        got = E.encode_host(X, cw, sq, Pt, 5, chunk=chunk)
        np.testing.assert_array_equal(got.cpu().numpy(), ref.cpu().numpy())
    enc = da.encode_dataset(book, X, beam_width=5, cross=cross)
    np.testing.assert_array_equal(enc.codes.astype(np.int64), ref.cpu().numpy().astype(np.int64))
    bad = X.copy()
    bad[1700, 3] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        E.encode_host(bad, cw, sq, Pt, 5, chunk=1000)
    with pytest.raises(ValueError, match="non-finite"):
        da.encode_dataset(book, bad, beam_width=5, cross=cross)


@pytest.mark.parametrize("M,D,n", [(8, 960, 1500), (3, 500, 300), (2, 256, 129)])
def test_wide_rows_d_tiled_table(M, D, n, monkeypatch):
    """D too wide for a resident tile image: the D-tiled tcgen05 table (streamed
    tf32 images, looser bound, band narrowing at L = 1) against the plain float64
    encoder -- default policy, forced on for every width, and forced off."""
    rng = np.random.default_rng(D + M)
    centers = rng.random((64, D)).astype(np.float32) * 0.3
    X = np.clip(centers[rng.integers(0, 64, n)] + 0.05 * rng.standard_normal((n, D)), 0, 1).astype(np.float32)
    cw = (rng.standard_normal((M, 256, D)) * (0.3 / np.arange(1, M + 1))[:, None, None]).astype(np.float32)
    cw[0] = np.abs(cw[0])
    book = da.Codebook(codewords=cw, order=np.arange(M))
    cross = cb.cross_products(book)
    cwd, sq = cb._codebook_dev(book)
    Pt, _ = cross.device()
    Xd = E.to_dev(X)
    for L in (1, 10):
        E.encode_config(1)
        plain = E.encode(Xd, cwd, sq, Pt, L)
        E.encode_config(0)
        for force in (None, "1", "0"):
            if force is None:
                monkeypatch.delenv("DA_TABLE_STREAM", raising=False)
            else:
                monkeypatch.setenv("DA_TABLE_STREAM", force)
            assert_same(E.encode(Xd, cwd, sq, Pt, L), plain)
        monkeypatch.delenv("DA_TABLE_STREAM", raising=False)
    # band narrowing on the resident-image table too (forced), and off at wide D
    for val in ("1", "0"):
        monkeypatch.setenv("DA_GREEDY_NARROW", val)
        E.encode_config(1)
        plain = E.encode(Xd, cwd, sq, Pt, 1)
        E.encode_config(0)
        assert_same(E.encode(Xd, cwd, sq, Pt, 1), plain)
    monkeypatch.delenv("DA_GREEDY_NARROW", raising=False)
