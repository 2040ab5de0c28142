"""Recheck counts per encoder mode on config-B-like data (vectors x stages)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E
import bench
n = 65536
X = E.to_dev(bench.rank_data(0, n))
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(X[:20000].contiguous(), cfg0)
Pt, sq = E.cross_full(cw)
sqe = E.einsum_sq(cw)
for L in (1, 10):
    for mode in (2, 3):
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        E.encode_config(mode, cnt)
        E.encode(X, cw, sqe, Pt, L, with_err=False)
        torch.cuda.synchronize()
        print(f"L={L} mode={mode} rechecks/vector={int(cnt.item()) / n:.1f}", flush=True)
E.encode_config(0)
