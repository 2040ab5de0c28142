"""Anneal pass over n rows (default: a 1/8 share of config B) with CUDA graphs on, timed with CUDA events,
plus the Lloyd-graph statistics.  usage: python tools/anneal_share.py [n] [reps]"""
import os, sys, json, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E, _native
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 125_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
X = E.to_dev(bench.rank_data(0, n))
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(X[:min(n, 100_000)].contiguous(), cfg0)
Pt, sq = E.cross_full(cw)
codes, _ = E.encode(X, cw, E.einsum_sq(cw), Pt, 10, out_dtype=torch.int32, with_err=False)
cfg1 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=1, rel_tol=0.0)
ts = []
for i in range(reps + 1):
    st = [cw.clone(), codes.clone(), Pt.clone(), sq.clone()]
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); E.da_sweep(X, *st, cfg1); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / 1e3)
g = (ctypes.c_longlong * 4)()
_native.load_library().da_lloyd_graph_stats(g)
print(json.dumps({"n": n, "pass_s": [round(t, 4) for t in ts], "graph_stats_eager_captured_replayed_failed": list(g)}))
