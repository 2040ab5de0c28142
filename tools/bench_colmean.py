"""Time the sequential-chain column mean (numpy X.mean(axis=0) order) on 1M x 128 f64."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_05194_b200 import _engine as E
X = torch.randn((1_000_000, 128), dtype=torch.float64, device="cuda")
m = torch.empty(128, dtype=torch.float64, device="cuda")
for _ in range(2):
    E.native.da_col_mean(E.P(X), 0, X.shape[0], 128, 128, E.P(m), E.stream())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    E.native.da_col_mean(E.P(X), 0, X.shape[0], 128, 128, E.P(m), E.stream())
e1.record(); torch.cuda.synchronize()
print(json.dumps({"col_mean_ms": e0.elapsed_time(e1) / 3}))
