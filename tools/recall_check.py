"""Recall@10 on config B: exhaustive ADC vs A-Tree (several l0) vs exact (GPU brute force)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E, atree as AT
from paper_1509_05194_b200.groundtruth import brute_force_knn
import bench
n = 1_000_000
X_h = bench.rank_data(0, n)
X = E.to_dev(X_h)
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(X[:100000].contiguous(), cfg0)
book = da.Codebook(codewords=cw.cpu().numpy(), order=np.arange(8))
cross = da.cross_products(book)
enc = da.encode_dataset(book, X_h, beam_width=10, cross=cross)
Q = bench.rank_data(7, 1000)
gt = brute_force_knn(X_h, Q, 10)
rec = lambda ids: float(np.mean([len(set(a) & set(b)) / 10.0 for a, b in zip(ids, gt.ids)]))
out = {}
eids, _ = da.exhaustive_adc_search_batch(book, enc, Q.astype(np.float64), 10, cross=cross)
out["exhaustive_adc"] = rec(eids)
eids100, _ = da.exhaustive_adc_search_batch(book, enc, Q.astype(np.float64), 100, cross=cross)
out["exhaustive_adc_recall10_at100"] = float(np.mean([len(set(a) & set(b)) / 10.0 for a, b in zip(eids100, gt.ids)]))
tree = AT.build_atree(enc, book, cross)
for l0 in (8, 32, 128):
    ids, _, _, _ = AT.atree_search_batch(tree, book, Q.astype(np.float64), AT.SearchParams(l0=l0, ls=2.0, r=10))
    out[f"atree_l0={l0}"] = rec(ids)
print(json.dumps(out))
