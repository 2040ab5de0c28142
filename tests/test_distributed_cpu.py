"""Row-sharded DA exchange steps, world_size 2 over gloo on CPU.

The device kernels produce per-shard partials; these tests feed the same
partials (computed with numpy) through the production merge code
(_engine._sharded_update, _engine._reseed_sharded, distributed.Comm) and
check the result against the unsharded reference semantics."""

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
