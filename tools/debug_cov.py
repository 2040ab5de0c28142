import os, sys
os.environ.setdefault("OPENBLAS_CORETYPE", "SkylakeX")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import cases
from paper_1509_05194_b200 import _engine as E
rng = np.random.default_rng(0)
for X64 in [cases.staged_case()["X"].astype(np.float64), rng.standard_normal((600, 12)), rng.standard_normal((600, 16)),
            rng.standard_normal((1500, 12)), rng.standard_normal((10000, 32)), rng.standard_normal((100, 12))]:
    n, D = X64.shape
    Xd = E.to_dev(X64)
    mean = torch.empty(D, dtype=torch.float64, device="cuda")
    E.native.da_col_mean(E.P(Xd), 0, n, D, D, E.P(mean), E.stream())
    cov = torch.empty((D, D), dtype=torch.float64, device="cuda")
    E.native.da_pca_cov(E.P(Xd), 0, n, D, D, E.P(mean), E.P(cov), 1, E.stream())
    mu = X64.mean(axis=0); Xc = X64 - mu
    ref = (Xc.T @ Xc) / (n - 1)
    got = cov.cpu().numpy()
    print(n, D, "mean eq", (mean.cpu().numpy() == mu).all(), "cov eq", (got == ref).mean(), np.abs(got - ref).max())
