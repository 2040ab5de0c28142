"""Row-sharded training end to end: several processes share the one visible
GPU and exchange through gloo (host-staged, so no kernel ever waits on another
process).  With the exact shard reductions (PCA ring, Lloyd leaf states) the
sharded run reproduces the one-GPU run -- and so the reference -- bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import cases
        import paper_1509_05194_b200 as da
        from paper_1509_05194_b200 import _engine as E
        from paper_1509_05194_b200 import distributed as D

        c = cases.train_case()
        X = c["X"]
        sl = D.shard_rows(len(X), world, rank)
        comm = D.Comm()
        cfg = da.TrainConfig(**c["config"])
        cw, codes, rep = D.train_from_scratch_sharded(E.to_dev(X[sl]), cfg, comm)
        q.put((rank, (cw.cpu().numpy(), codes.cpu().numpy(), rep.distortions())))
    except Exception as e:
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_shards_on_one_gpu():
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import cases
    import paper_1509_05194_b200 as da

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert not isinstance(out[0], str), out[0]
    assert not isinstance(out[1], str), out[1]
    cw0, codes0, d0 = out[0]
    cw1, codes1, d1 = out[1]
    np.testing.assert_array_equal(cw0, cw1)  # replicated state stays identical
    np.testing.assert_array_equal(d0, d1)
    assert (np.diff(d0) <= 1e-6 * d0[:-1]).all()
    c = cases.train_case()
    _, _, rep = da.train_from_scratch(c["X"], da.TrainConfig(**c["config"]))
    single = rep.distortions()
    # exact shard reductions: the one-GPU run's codebook; distortions are
    # per-shard sums allreduced (last-bit differences only)
    np.testing.assert_allclose(d0, single, rtol=1e-12)


@pytest.fixture(scope="module")
def gloo1():
    """A one-process gloo group for the world-1 equivalence tests."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), DA_SHARD_LOOP="1")
    dist.init_process_group("gloo", rank=0, world_size=1)
    yield
    dist.destroy_process_group()
    os.environ.pop("DA_SHARD_LOOP", None)


@pytest.mark.parametrize("K,active,seed", [(8, 3, 0), (64, 5, 1), (200, 2, 2)])
def test_sharded_lloyd_world1_equals_single(gloo1, K, active, seed):
    """One shard: the pipelined sharded Lloyd loop (two collectives per
    iteration, active-prefix sums, speculative next iteration, reseeds) must
    give the one-GPU loop's centroids, labels and trace bit for bit.  K=200 on
    clustered data empties clusters, so the reseed path runs."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import cases
    from paper_1509_05194_b200 import _engine as E
    from paper_1509_05194_b200 import distributed as D

    X = cases.mixture(3000, 9, 6, 0.05, 40 + seed).astype(np.float64)
    rng = np.random.default_rng(seed)
    C0 = X[rng.choice(len(X), K, replace=False)].copy()
    Xd, Cd = E.to_dev(X), E.to_dev(C0)
    comm = D.Comm().bind_rows(len(X))
    C1, l1, t1 = E.lloyd(Xd, Cd, active, 30, None)
    C2, l2, t2 = E.lloyd(Xd, Cd, active, 30, comm)
    assert torch.equal(C1, C2)
    assert torch.equal(l1, l2)
    assert t1 == t2


def test_sharded_sweep_world1_equals_single(gloo1):
    """A full da_sweep through the sharded engine on one shard (PCA, staged
    Lloyd, beam re-encode) equals the one-GPU sweep bit for bit."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import cases
    import paper_1509_05194_b200 as da
    from paper_1509_05194_b200 import _engine as E
    from paper_1509_05194_b200 import distributed as D

    c = cases.train_case()
    X = E.to_dev(c["X"])
    cfg = da.TrainConfig(**{**c["config"], "sweeps": 0})
    cw, codes = E.growth_pass(X, cfg)
    Pt, sq = E.cross_full(cw)
    st1 = [cw.clone(), codes.clone(), Pt.clone(), sq.clone()]
    st2 = [cw.clone(), codes.clone(), Pt.clone(), sq.clone()]
    cfg1 = da.TrainConfig(**{**c["config"], "sweeps": 1, "rel_tol": 0.0})
    E.da_sweep(X, *st1, cfg1)
    D.da_sweep_sharded(X, *st2, cfg1, D.Comm())
    for a, b in zip(st1, st2):
        assert torch.equal(a, b)


def _config_a_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_1509_05194_b200 as da
        from paper_1509_05194_b200 import _engine as E
        from paper_1509_05194_b200 import distributed as D
        from paper_1509_05194_b200 import synthetic

        X = synthetic.config_a()
        sl = D.shard_rows(len(X), world, rank)
        cfg = da.TrainConfig(m_count=4, k_count=256, beam_width=10, sweeps=3, rel_tol=0.0)
        cw, codes, rep = D.train_from_scratch_sharded(E.to_dev(X[sl]), cfg, D.Comm())
        q.put((rank, (cw.cpu().numpy(), codes.cpu().numpy(), rep.distortions())))
    except Exception as e:
        import traceback

        q.put((rank, traceback.format_exc() + repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_config_a_sharded_matches_reference(world, golden):
    """BASELINE config A trained over `world` row shards (gloo, one GPU) against
    the reference's own 16-step run, at the north-star bar: dictionaries within
    1e-4 relative Frobenius per m, MSE within 1e-4, codes equal except where the
    oracle's decision gap is below 1e-6.  The PCA moments are bit-identical by
    construction (the ring of distributed.exact_pca_moments); only the Lloyd
    sums are added in another order (shard partials, allreduced)."""
    import paper_1509_05194_b200 as da
    from oracle import da_oracle as O
    from paper_1509_05194_b200 import codebook as cb
    from paper_1509_05194_b200 import synthetic

    g = golden("config_a.npz")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_config_a_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=900) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(out[r], str), out[r]
    cw0 = out[0][0]
    for r in range(1, world):
        np.testing.assert_array_equal(out[r][0], cw0)      # replicas identical
        np.testing.assert_array_equal(out[r][2], out[0][2])
    book, perm = cb.reorder_by_variance(da.Codebook(codewords=cw0, order=np.arange(4, dtype=np.int64)))
    np.testing.assert_array_equal(book.order, g["order"])
    ref = g["cw"].astype(np.float64)
    got = book.codewords.astype(np.float64)
    for m in range(4):
        rel = np.linalg.norm(got[m] - ref[m]) / np.linalg.norm(ref[m])
        print(f"world {world} dictionary {m}: rel Frobenius {rel:.3e}, "
              f"{int((book.codewords[m] != g['cw'][m]).sum())} entries differ")
        assert rel <= 1e-4, (m, rel)
    dist_ = np.asarray(out[0][2])
    np.testing.assert_allclose(dist_, g["dist"], rtol=1e-4)
    codes = np.concatenate([out[r][1] for r in range(world)])[:, perm]
    diff = np.flatnonzero((codes != g["codes"]).any(axis=1))
    if diff.size:
        X = synthetic.config_a()
        P, _ = O.cross_table(g["cw"])
        gap = O.beam_min_gap(g["cw"].astype(np.float64), P, X[diff].astype(np.float64), 10)
        assert (gap < 1e-6).all(), (diff[:10], gap[:10])
    mse = cb.distortion(book, synthetic.config_a(), da.EncodedDataset(codes.astype(np.uint8), 256))
    assert abs(mse - float(g["mse"])) <= 1e-4 * float(g["mse"]), (mse, float(g["mse"]))
    # what the exact shard reductions actually deliver: the reference's bits
    np.testing.assert_array_equal(book.codewords, g["cw"])
    np.testing.assert_array_equal(codes, g["codes"])


def _lloyd_worker(rank, world, port, layout, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import cases
        from paper_1509_05194_b200 import _engine as E
        from paper_1509_05194_b200 import distributed as D

        res = []
        for K, active, seed in [(8, 3, 0), (64, 5, 1), (200, 2, 2), (37, 9, 3)]:
            X = cases.mixture(3000, 9, 6, 0.05, 40 + seed).astype(np.float64)
            rng = np.random.default_rng(seed)
            C0 = X[rng.choice(len(X), K, replace=False)].copy()
            lo = sum(layout[:rank])
            Xs = E.to_dev(X[lo:lo + layout[rank]])
            comm = D.Comm().bind_rows(layout[rank])
            for lazy in (False, True):
                C2, l2, t2 = E.lloyd(Xs, E.to_dev(C0), active, 30, comm, want_trace=not lazy)
                res.append((C2.cpu().numpy(), l2.cpu().numpy(), t2))
        q.put((rank, res))
    except Exception:
        import traceback

        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("layout,rounds", [([1500, 1500], None), ([5, 2990, 5], None), ([1000, 0, 1200, 800], None),
                                           ([2999, 1], None), ([5, 2990, 5], "1"), ([1000, 0, 1200, 800], "1")])
def test_exact_sharded_lloyd_equals_one_gpu(layout, rounds, monkeypatch):
    """The exact sharded Lloyd update (da_gs_shard_*: leaf states handed across
    shard boundaries, W-1 neighbour rounds, one leaf-sum allreduce) gives the
    one-GPU centroids and labels bit for bit on every shard layout, including
    tiny and empty shards (a leaf crossing several shards) and reseeds (K=200).
    rounds="1": one neighbour round per update, so leaves crossing two or more
    boundaries trip the overflow flag and the update is redone with world-1
    rounds -- same bits."""
    if rounds is not None:
        monkeypatch.setenv("DA_SHARD_ROUNDS", rounds)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import cases
    from paper_1509_05194_b200 import _engine as E

    world = len(layout)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_lloyd_worker, args=(r, world, port, layout, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(out[r], str), out[r]
    i = 0
    for K, active, seed in [(8, 3, 0), (64, 5, 1), (200, 2, 2), (37, 9, 3)]:
        X = cases.mixture(3000, 9, 6, 0.05, 40 + seed).astype(np.float64)
        rng = np.random.default_rng(seed)
        C0 = X[rng.choice(len(X), K, replace=False)].copy()
        for lazy in (False, True):
            C1, l1, t1 = E.lloyd(E.to_dev(X), E.to_dev(C0), active, 30, None, want_trace=not lazy)
            for r in range(world):
                np.testing.assert_array_equal(out[r][i][0], C1.cpu().numpy(), err_msg=f"K={K} rank {r} lazy={lazy}")
            labels = np.concatenate([out[r][i][1] for r in range(world)])
            np.testing.assert_array_equal(labels, l1.cpu().numpy())
            if not lazy:
                assert len(out[0][i][2]) == len(t1)
                np.testing.assert_allclose(out[0][i][2], t1, rtol=1e-13)
            i += 1


def _online_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_1509_05194_b200 as da
        from paper_1509_05194_b200 import codebook as cb
        from paper_1509_05194_b200 import distributed as D
        from paper_1509_05194_b200 import synthetic

        chunks = [synthetic.mixture_b_chunk(3, c, n=3000).astype(np.uint8) for c in range(3)]
        cfg0 = da.TrainConfig(m_count=4, k_count=32, beam_width=4, sweeps=0, rel_tol=0.0)
        book, _, _ = da.train_from_scratch(chunks[0].astype(np.float32), cfg0)
        cw0, _ = cb._codebook_dev(book)
        cfg = da.TrainConfig(m_count=4, k_count=32, beam_width=4, sweeps=1, rel_tol=0.0)
        mine = [ch[D.shard_rows(len(ch), world, rank)] for ch in chunks[1:]]
        cw, reps = D.train_online_stream(cw0, mine, cfg, D.Comm())
        q.put((rank, (cw.cpu().numpy(), [r.distortions() for r in reps])))
    except Exception:
        import traceback

        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_online_stream_sharded_equals_one_gpu(world):
    """Config-D style online DA: uint8 chunks, each rank streaming its slice
    through pinned async uploads (ChunkFeeder) into train_online_sharded; the
    codebook after every chunk equals the one-GPU train_online on the whole chunk."""
    import paper_1509_05194_b200 as da
    from paper_1509_05194_b200 import synthetic

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_online_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(out[r], str), out[r]
        np.testing.assert_array_equal(out[r][0], out[0][0])
    chunks = [synthetic.mixture_b_chunk(3, c, n=3000).astype(np.uint8) for c in range(3)]
    cfg0 = da.TrainConfig(m_count=4, k_count=32, beam_width=4, sweeps=0, rel_tol=0.0)
    book, _, _ = da.train_from_scratch(chunks[0].astype(np.float32), cfg0)
    cfg = da.TrainConfig(m_count=4, k_count=32, beam_width=4, sweeps=1, rel_tol=0.0)
    for c in chunks[1:]:
        book, rep = da.train_online(book, c.astype(np.float32), cfg)
    np.testing.assert_array_equal(out[0][0], book.codewords)
    np.testing.assert_allclose(out[0][1][-1], rep.distortions(), rtol=1e-12)
