"""Row-sharded DA exchange steps, world_size 2 over gloo on CPU.

The device kernels produce per-shard partials; these tests feed the same
partials (computed with numpy) through the production merge code
(_engine._sharded_update, _engine._reseed_sharded, distributed.Comm) and
check the result against the unsharded reference semantics."""

import functools
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1509_05194_b200 import _engine as E
from paper_1509_05194_b200 import distributed as D


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # surface failures to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return out


def dataset():
    rng = np.random.default_rng(0)
    X = rng.standard_normal((1001, 6)) * 10.0 ** rng.uniform(-1, 1, 6)
    lab = rng.integers(0, 9, 1001)
    lab[lab == 4] = 5  # label 4 empty
    errs = rng.uniform(0, 1, 1001)
    errs[[17, 600, 900]] = 5.0  # tie at the top: higher global row id wins
    return X, lab, errs


def _update_case(rank, world):
    X, lab, _ = dataset()
    sl = D.shard_rows(len(X), world, rank)
    comm = D.Comm().bind_rows(sl.stop - sl.start)
    K = 10
    sums = np.zeros((K, X.shape[1]))
    np.add.at(sums, lab[sl], X[sl])
    counts = np.bincount(lab[sl], minlength=K).astype(np.int32)
    C = torch.full((K, X.shape[1]), -3.0, dtype=torch.float64)
    red = torch.from_numpy(np.concatenate([sums.ravel(), counts.astype(np.float64)]))
    n_empty = int(E._sharded_update(red, K, X.shape[1], C, comm))
    cnt = red[K * X.shape[1]:].numpy().astype(np.int64)
    assert n_empty == int((cnt == 0).sum())
    return cnt.tolist(), C.numpy().tolist(), comm.row_offset, comm.total(sl.stop - sl.start)


def test_sharded_update_matches_unsharded_means():
    out = run(_update_case)
    X, lab, _ = dataset()
    K = 10
    cnt_ref = np.bincount(lab, minlength=K)
    sums = np.zeros((K, X.shape[1]))
    np.add.at(sums, lab, X)
    for rank in (0, 1):
        cnt, C, off, total = out[rank]
        assert total == len(X)
        assert off == (0 if rank == 0 else D.shard_rows(len(X), 2, 0).stop)
        np.testing.assert_array_equal(cnt, cnt_ref)
        C = np.array(C)
        filled = cnt_ref > 0
        np.testing.assert_allclose(C[filled], sums[filled] / cnt_ref[filled, None], rtol=1e-13)
        assert (C[~filled] == -3.0).all()  # empties left for the reseed
    np.testing.assert_array_equal(np.array(out[0][1]), np.array(out[1][1]))  # replicas agree


def _reseed_case(rank, world):
    X, _, errs = dataset()
    sl = D.shard_rows(len(X), world, rank)
    comm = D.Comm().bind_rows(sl.stop - sl.start)
    empty = [1, 4, 7, 8]
    C = torch.zeros((10, X.shape[1]), dtype=torch.float64)
    E._reseed_sharded(torch.from_numpy(X[sl].copy()), torch.from_numpy(errs[sl].copy()), np.array(empty), C, comm)
    return C.numpy().tolist()


def test_sharded_reseed_picks_the_global_worst_rows():
    out = run(_reseed_case)
    X, _, errs = dataset()
    worst = np.argsort(errs, kind="stable")[::-1][:4]  # annq/clustering.py:195
    assert list(worst[:3]) == [900, 600, 17]
    for rank in (0, 1):
        C = np.array(out[rank])
        np.testing.assert_array_equal(C[[1, 4, 7, 8]], X[worst])


def test_merge_worst_order():
    err = np.array([1.0, 3.0, 3.0, -np.inf, 2.0])
    gid = np.array([10, 4, 7, -1, 2])
    np.testing.assert_array_equal(D.merge_worst(err, gid, 3), [2, 1, 4])


@pytest.mark.parametrize("n,world", [(10, 3), (1000, 8), (7, 8)])
def test_shard_rows_partition(n, world):
    parts = [D.shard_rows(n, world, r) for r in range(world)]
    assert parts[0].start == 0 and parts[-1].stop == n
    for a, b in zip(parts, parts[1:]):
        assert a.stop == b.start
    sizes = [p.stop - p.start for p in parts]
    assert max(sizes) - min(sizes) <= 1


# ---------------------------------------------------------------------------
# sharded PCA ring (distributed.exact_pca_moments): the chains must be cut and
# continued so that every shard layout gives the one-shard bits.


class _NumpyPcaOps:
    """Host stand-in for the device kernels: the same dependency structure
    (one add chain per column, one accumulation chain per cov block, block
    totals added in order), plain float64 multiply + add.  Any reordering of
    those chains across a shard boundary changes the bits."""

    def zeros(self, shape):
        return torch.zeros(shape, dtype=torch.float64)

    def div(self, t, d):
        return t / torch.full_like(t, float(d))

    def col_sums(self, X, init):
        s = init.clone() if init is not None else torch.zeros(X.shape[1], dtype=torch.float64)
        for r in range(X.shape[0]):
            s = s + X[r]
        return s

    def cov_chains(self, X, mean, starts, init):
        out = []
        for i in range(len(starts) - 1):
            acc = init.clone() if (i == 0 and init is not None) else torch.zeros((X.shape[1],) * 2, dtype=torch.float64)
            for r in range(starts[i], starts[i + 1]):
                xc = X[r] - mean
                acc = acc + torch.outer(xc, xc)
            out.append(acc)
        return torch.stack(out)

    def fold(self, total, parts):
        s = total.clone() if total is not None else parts[0].clone()
        for p in parts[(0 if total is not None else 1):]:
            s = s + p
        return s


class _OneShard:
    rank, world = 0, 1

    def sizes(self, n):
        return [n]

    def broadcast_(self, t, src):
        return t


def _ring_data():
    rng = np.random.default_rng(7)
    return torch.from_numpy(rng.standard_normal((1000, 5)) * 10.0 ** rng.uniform(-2, 3, 5))


RING_LAYOUTS = [[500, 500], [100, 200, 700], [0, 1000, 0], [384, 308, 308], [383, 2, 615], [1, 999]]


def _ring_fn(layout, rank, world):
    X = _ring_data()
    lo = sum(layout[:rank])
    comm = D.Comm()
    comm.bind_rows(layout[rank])
    mean, cov = D.exact_pca_moments(X[lo:lo + layout[rank]], comm, _NumpyPcaOps())
    return mean.numpy(), cov.numpy()


@pytest.mark.parametrize("layout", RING_LAYOUTS)
def test_exact_pca_ring_equals_one_shard(layout):
    X = _ring_data()
    m1, c1 = D.exact_pca_moments(X, _OneShard(), _NumpyPcaOps())
    # the column chains are numpy's own X.mean(axis=0) order
    np.testing.assert_array_equal(m1.numpy(), X.numpy().mean(axis=0))
    out = run(functools.partial(_ring_fn, layout), world=len(layout))
    for r in range(len(layout)):
        assert not isinstance(out[r], str), out[r]
        np.testing.assert_array_equal(out[r][0], m1.numpy())
        np.testing.assert_array_equal(out[r][1], c1.numpy())


def test_cov_segments_cover_the_blocks():
    st = D.blas_block_starts(1000)
    assert st == [0, 384, 692, 1000]
    segs, cf, ol, tv = D.cov_segments(1000, 100, 300)
    assert segs == [(0, 200)] and cf and ol and not tv
    segs, cf, ol, tv = D.cov_segments(1000, 384, 1000)
    assert segs == [(0, 308), (308, 616)] and not cf and not ol and tv
    for n in (1, 383, 384, 385, 767, 768, 769, 5000):
        st = D.blas_block_starts(n)
        assert st[-1] == n and all(0 < b - a <= 384 for a, b in zip(st[:-1], st[1:]))


def _shift_fn(rank, world):
    comm = D.Comm()
    send = torch.full((5,), float(rank + 1), dtype=torch.float64)
    recv = torch.full((5,), -1.0, dtype=torch.float64)
    comm.shift_(send, recv)
    return recv.numpy()


@pytest.mark.parametrize("world", [2, 3])
def test_shift_passes_right(world):
    """Comm.shift_: every rank sends to rank+1 and receives from rank-1 in one
    batched exchange (the exact shard reductions' neighbour rounds); rank 0's
    receive buffer is untouched."""
    out = run(_shift_fn, world=world)
    np.testing.assert_array_equal(out[0], np.full(5, -1.0))
    for r in range(1, world):
        np.testing.assert_array_equal(out[r], np.full(5, float(r)))
