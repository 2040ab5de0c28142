import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E
from paper_1509_05194_b200 import codebook as cb
L = int(sys.argv[1]) if len(sys.argv) > 1 else 16
rng = np.random.default_rng(L)
for M, K, D in [(3, 8, 6), (4, 16, 17), (2, 300, 9), (8, 256, 128)]:
    book = da.Codebook(codewords=rng.standard_normal((M, K, D)).astype(np.float32), order=np.arange(M))
    X = rng.standard_normal((700, D)).astype(np.float32)
    cross = cb.cross_products(book)
    cw, sq = cb._codebook_dev(book)
    Pt, _ = cross.device()
    Xd = E.to_dev(X)
    print(M, K, D, flush=True)
    E.encode_config(3)
    tc = E.encode(Xd, cw, sq, Pt, L)
    torch.cuda.synchronize()
    E.encode_config(1)
    pl = E.encode(Xd, cw, sq, Pt, L)
    print("same", bool((tc[0] == pl[0]).all()), flush=True)
