"""Encode time per beam width for the gather filter (mode 2) and the tcgen05 filter (mode 3)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
X = E.to_dev(bench.rank_data(0, n))
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(X[:100000].contiguous(), cfg0)
Pt, sq = E.cross_full(cw)
sqe = E.einsum_sq(cw)
for L in (1, 2, 4, 6, 8, 10, 16, 32):
    row = []
    for mode in (2, 3):
        E.encode_config(mode)
        E.encode(X, cw, sqe, Pt, L, with_err=False)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(2):
            t0 = time.perf_counter()
            E.encode(X, cw, sqe, Pt, L, with_err=False)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        row.append(best)
    print(f"L={L:3d} gather {row[0]*1e3:8.1f} ms  tc {row[1]*1e3:8.1f} ms", flush=True)
E.encode_config(0)
