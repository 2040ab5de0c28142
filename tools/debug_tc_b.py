import os, sys
os.environ["DA_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E
import bench
X = E.to_dev(bench.rank_data(0, 20000))
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(X[:10000].contiguous(), cfg0)
Pt, sq = E.cross_full(cw)
sqe = E.einsum_sq(cw)
for L in (1, 2, 10):
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    E.encode_config(0, cnt)
    c0, e0 = E.encode(X, cw, sqe, Pt, L)
    torch.cuda.synchronize()
    E.encode_config(1)
    c1, e1 = E.encode(X, cw, sqe, Pt, L)
    print("L", L, "rechecked", int(cnt.item()), "mismatch", int((c0 != c1).any(dim=1).sum().item()), flush=True)
E.encode_config(0)
