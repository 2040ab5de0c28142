import os, sys
os.environ.setdefault("OPENBLAS_CORETYPE", "SkylakeX")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import cases
from paper_1509_05194_b200 import _engine as E
from oracle import da_oracle as O
c = cases.staged_case()
X64 = c["X"].astype(np.float64)
Xd = E.to_dev(X64)
R, mu, var, Rh = E.pca(Xd)
Ro, muo = O.pca(X64)
print("mean eq", (mu.cpu().numpy() == muo).all(), "R eq", (Rh == Ro).all(), np.abs(Rh - Ro).max())
Xr = E.rotate(Xd, R, mu).cpu().numpy()
Xro = (X64 - muo) @ Ro.T
print("Xr eq", (Xr == Xro).mean())
C0 = c["C"]
Cr = E.rotate(E.to_dev(C0), R, mu).cpu().numpy()
Cro = (C0 - muo) @ Ro.T
print("Cr eq", (Cr == Cro).mean())
Cg, Co = E.to_dev(Cro), Cro
for dims in O.schedule(12):
    a, la, ta = E.lloyd(E.to_dev(Xro), Cg, dims, 30)
    b, lb, tb = O.lloyd(Xro, Co, dims, 30)
    print(dims, "C eq", (a.cpu().numpy() == b).mean(), "lab eq", (la.cpu().numpy() == lb).mean(), "trace eq", ta == tb)
    Cg, Co = E.to_dev(b), b
Cinv = E.rotate(E.to_dev(Co), R, mu, inverse=True).cpu().numpy()
print("inverse eq", (Cinv == Co @ Ro + muo).mean())
