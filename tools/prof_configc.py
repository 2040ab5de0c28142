"""Encode 65536 config-C (D=960) vectors once at a chosen beam width (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E, synthetic
L = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
X = E.to_dev(np.ascontiguousarray(synthetic.config_c(n=n), dtype=np.float32))
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(X[:20000].contiguous(), cfg0)
Pt, _ = E.cross_full(cw)
sqe = E.einsum_sq(cw)
E.encode(X, cw, sqe, Pt, L, with_err=False)
torch.cuda.synchronize()
print("ok")
