"""Gather filter (mode 2) timing on config B against the tcgen05 filter (mode 3)
as the identity check: codes and errors must be identical."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
Ls = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [4, 10, 16]
X = E.to_dev(bench.rank_data(0, n))
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(X[:100000].contiguous(), cfg0)
Pt, sq = E.cross_full(cw)
sqe = E.einsum_sq(cw)
for L in Ls:
    res = {}
    for mode in (3, 2):
        E.encode_config(mode)
        out = E.encode(X, cw, sqe, Pt, L)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            E.encode(X, cw, sqe, Pt, L, with_err=False)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        res[mode] = (best, out)
    same = all(torch.equal(a, b) for a, b in zip(res[3][1], res[2][1]))
    print(f"L={L:3d} gather {res[2][0]*1e3:8.1f} ms  tcgen05 {res[3][0]*1e3:8.1f} ms  identical={same}", flush=True)
E.encode_config(0)
