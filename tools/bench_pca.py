import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_05194_b200 import _engine as E, _native
import bench
X = E.to_dev(bench.rank_data(0, 1_000_000))
for rep in range(2):
    _native.prof_enable(True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    R, mean, _, _ = E.pca(X)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    _native.prof_enable(False)
    print(json.dumps({"pca_s": dt, "kernels": _native.prof_collect()}))
mu = X.double().mean(dim=0)
print("mean max diff vs torch", (mean - mu).abs().max().item())
