import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E, codebook as cb
rng = np.random.default_rng(10)
for (M, K, D, n) in [(3, 8, 6, 50), (2, 8, 6, 50), (3, 16, 6, 50), (3, 8, 32, 50)]:
    book = da.Codebook(codewords=rng.standard_normal((M, K, D)).astype(np.float32), order=np.arange(M))
    X = rng.standard_normal((n, D)).astype(np.float32)
    cross = cb.cross_products(book); cw, sq = cb._codebook_dev(book); Pt, _ = cross.device(); Xd = E.to_dev(X)
    bad = []
    for L in [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 16]:
        E.encode_config(0); t = E.encode(Xd, cw, sq, Pt, L)
        E.encode_config(1); p = E.encode(Xd, cw, sq, Pt, L)
        tc, pc = t[0].cpu().numpy(), p[0].cpu().numpy()
        mism = np.flatnonzero((tc != pc).any(axis=1))
        if mism.size: bad.append((L, mism.size, mism[:5].tolist(), tc[mism[0]].tolist(), pc[mism[0]].tolist()))
    print((M, K, D), bad)
E.encode_config(0)
