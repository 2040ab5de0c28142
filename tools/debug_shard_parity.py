"""Where does a sharded run first differ from the one-GPU run?  2 ranks over
gloo on one GPU: PCA moments, one Lloyd call, one growth step."""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1509_05194_b200 as da
    from paper_1509_05194_b200 import _engine as E, distributed as D, synthetic
    X = synthetic.config_a()
    sl = D.shard_rows(len(X), world, rank)
    comm = D.Comm().bind_rows(sl.stop - sl.start)
    Xd = E.to_dev(X)
    Xs = E.to_dev(X[sl])
    R1, m1, v1, _ = E.pca(Xd)
    R2, m2, v2, _ = E.pca(Xs, comm)
    if rank == 0:
        print("pca mean equal", torch.equal(m1, m2), "R equal", torch.equal(R1, R2), flush=True)
    # one lloyd call on rotated data
    Xr1 = E.rotate(Xd, R1, m1)
    Xr2 = E.rotate(Xs, R1, m1)
    rng = np.random.default_rng(0)
    C0 = E.to_dev(X[rng.choice(len(X), 256, replace=False)].astype(np.float64))
    C0r = E.rotate(C0, R1, m1)
    for act in (2, 3, 32):
        for lazy in (False, True):
            Ca, la, ta = E.lloyd(Xr1, C0r, act, 30, None, want_trace=not lazy)
            Cb, lb, tb = E.lloyd(Xr2, C0r, act, 30, comm, want_trace=not lazy)
            lb_all = comm.allgather(lb.to(torch.int64)).cpu()
            if rank == 0:
                d = (Ca - Cb).abs().max().item()
                print(f"lloyd act={act} lazy={lazy}: C maxdiff {d:.3e}, labels diff {(la.cpu().to(torch.int64) != lb_all).sum().item()}, "
                      f"iters {len(ta)} {len(tb)} trace0 {ta[:2]} {tb[:2]}", flush=True)
    # growth step by step
    cfg = da.TrainConfig(m_count=4, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
    cw1, c1 = E.growth_pass(Xd, cfg)
    cw2, c2 = E.growth_pass(Xs, cfg, comm=comm)
    if rank == 0:
        for m in range(4):
            print("growth m", m, "cw maxdiff", (cw1[m] - cw2[m]).abs().max().item(), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    import socket
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mp.spawn(worker, args=(2, port), nprocs=2)
