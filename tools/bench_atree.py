"""A-Tree over config-B codes: GPU build time (vs the host oracle build), GPU batched search throughput.
usage: python tools/bench_atree.py [n] [nq]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E, atree as AT
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000
X = E.to_dev(bench.rank_data(0, n))
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(X[:100000].contiguous(), cfg0)
book = da.Codebook(codewords=cw.cpu().numpy(), order=np.arange(8))
cross = da.cross_products(book)
Pt, _ = cross.device()
sq = E.einsum_sq(cw)
codes, _ = E.encode(X, cw, sq, Pt, 10, out_dtype=torch.uint8, with_err=False)
enc = da.EncodedDataset(codes=codes.cpu().numpy(), k_count=256, codebook_hash=book.content_hash())
AT.build_atree(enc, book, cross)                # warm-up (scratch growth)
torch.cuda.synchronize()
t0 = time.perf_counter()
tree = AT.build_atree(enc, book, cross)
t_build = time.perf_counter() - t0
from oracle.atree_build import build_atree_host   # the host restatement, timed for comparison
t0 = time.perf_counter()
tree_h = build_atree_host(enc, book, cross)
t_host = time.perf_counter() - t0
same = all(np.array_equal(getattr(tree, f), getattr(tree_h, f)) for f in AT._TREE_FIELDS)
Q = bench.rank_data(7, nq).astype(np.float64)
out = {"n": n, "nq": nq, "build_s_gpu": t_build, "build_s_host_oracle": t_host, "same_arrays": same, "nodes": tree.node_count, "leaves": tree.leaf_count}
for l0 in (8, 32):
    params = AT.SearchParams(l0=l0, ls=2.0, r=10)
    AT.atree_search_batch(tree, book, Q, params)   # warm-up sizes the per-CTA scratch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ids, d, cnt, st = AT.atree_search_batch(tree, book, Q, params)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out[f"l0={l0}"] = {"queries_per_s": nq / dt, "ms": dt * 1e3, "mean_nodes_visited": float(st[:, 0].mean())}
print(json.dumps(out))
