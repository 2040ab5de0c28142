"""Time one anneal pass through the row-sharded (NCCL) engine against the
single-GPU engine on the same config-B data, and check that at world 1 they
give the same dictionaries and codes.

usage: python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 \
           --master-port 29511 tools/bench_anneal_sharded.py [n]
"""
import os, sys, time, json
os.environ.setdefault("DA_SHARD_LOOP", "1")   # time the shard loop even at world 1
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import torch.distributed as dist
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E, distributed as DD
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
dist.init_process_group("nccl")
X = E.to_dev(bench.rank_data(rank, n))
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(X[:100_000].contiguous(), cfg0)
Pt, sq = E.cross_full(cw)
codes, _ = E.encode(X, cw, E.einsum_sq(cw), Pt, 10, out_dtype=torch.int32, with_err=False)
cfg1 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=1, rel_tol=0.0)
comm = DD.Comm()
fast = DD.Comm(exact=False)


def run(sharded):
    state = [cw.clone(), codes.clone(), Pt.clone(), sq.clone()]
    rep = da.TrainReport(config=cfg1)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if sharded:
        DD.da_sweep_sharded(X, *state, cfg1, sharded, report=rep)
    else:
        E.da_sweep(X, *state, cfg1, report=rep)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, state, rep


run(comm)  # warm-up (scratch growth, NCCL setup)
run(fast)
ts, ss, rs = run(comm)
tf, sf, rf = run(fast)
t1, s1, r1 = None, None, None
if dist.get_world_size() == 1:
    run(False)
    t1, s1, r1 = run(False)
if rank == 0:
    out = {"n": n, "world": dist.get_world_size(), "sharded_exact_s": ts, "sharded_fast_s": tf, "single_s": t1,
           "exact_per_dict": [round(s.seconds, 3) for s in rs.steps],
           "fast_per_dict": [round(s.seconds, 3) for s in rf.steps]}
    if s1 is not None:
        out.update({"exact_same_codewords": bool(torch.equal(ss[0], s1[0])),
                    "exact_same_codes": bool(torch.equal(ss[1], s1[1])),
                    "fast_same_codewords": bool(torch.equal(sf[0], s1[0])),
                    "single_per_dict": [round(s.seconds, 3) for s in r1.steps]})
    print(json.dumps(out))
dist.destroy_process_group()
