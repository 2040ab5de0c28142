"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): encode (greedy L=1, pair L=4, lean L=10,
tcgen05 filter), tcgen05 score table, assign (tcgen05 + recheck, small-d),
group sums (one GPU and the sharded leaf-state path at world 1), PCA, ADC,
A-Tree search.  usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E, codebook as cb
import bench

X = bench.rank_data(0, 3000)
cfg = da.TrainConfig(m_count=4, k_count=64, beam_width=4, sweeps=1, rel_tol=0.0)
book, enc, rep = da.train_from_scratch(X, cfg)          # growth + sweep: PCA, Lloyd, group sums, assigns, encode
cross = cb.cross_products(book)
for L in (1, 4, 10):
    da.encode_dataset(book, X[:512], beam_width=L, cross=cross)
E.encode_config(3)
da.encode_dataset(book, X[:256], beam_width=10, cross=cross)   # tcgen05 residual-GEMM filter
E.encode_config(0)
cfg8 = da.TrainConfig(m_count=2, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
b8, e8, _ = da.train_from_scratch(X, cfg8)                 # K=256: tcgen05 assign + table paths
da.encode_dataset(b8, X[:300], beam_width=10)
q = X[5].astype(np.float64)
da.exhaustive_adc_search(b8, e8, q, 10)
from paper_1509_05194_b200 import atree as AT
tree = AT.build_atree(e8, b8, cb.cross_products(b8))
AT.atree_search(tree, b8, q, AT.SearchParams(l0=2, ls=2.0, r=5))
torch.cuda.synchronize()
print("sanitize run ok")
