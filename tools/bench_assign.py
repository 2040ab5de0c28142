"""Time the assign kernels (tensor-core vs float64) on config-B-like rotated data."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_05194_b200 import _engine as E
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
dims = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 8, 32, 128]
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((n, 128), dtype=torch.float64, device="cuda", generator=g) * 30
C = X[torch.randint(0, n, (256,), device="cuda", generator=g)] + torch.randn((256, 128), dtype=torch.float64, device="cuda", generator=g)
out = {}
for d in dims:
    xx = E.row_sqnorms(X, d)
    cc = E.row_sqnorms(C, d)
    for mode in (0, 1):
        E.assign_config(mode)
        for _ in range(2):
            E.assign(X, d, C, cc=cc, xx=xx)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 5
        for _ in range(reps):
            E.assign(X, d, C, cc=cc, xx=xx)
        e1.record(); torch.cuda.synchronize()
        out[f"d={d} {'tc' if mode == 0 else 'f64'}"] = round(e0.elapsed_time(e1) / reps, 3)
E.assign_config(0)
print(json.dumps({"n": n, "ms_per_assign": out}))
