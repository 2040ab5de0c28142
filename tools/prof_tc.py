"""Encode 65536 config-B vectors once with a chosen encoder mode (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E
import bench
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 3
L = int(sys.argv[2]) if len(sys.argv) > 2 else 10
X = E.to_dev(bench.rank_data(0, 65536))
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(X[:20000].contiguous(), cfg0)
Pt, sq = E.cross_full(cw)
sqe = E.einsum_sq(cw)
E.encode_config(mode)
E.encode(X, cw, sqe, Pt, L, with_err=False)
torch.cuda.synchronize()
print("ok")
