"""Time one full anneal pass (da_sweep over M dictionaries) on config B with a
per-kernel breakdown.  usage: python tools/bench_anneal.py [n]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E, _native
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
X = E.to_dev(bench.rank_data(0, n))
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(X[:100_000].contiguous(), cfg0)
Pt, sq = E.cross_full(cw)
codes, _ = E.encode(X, cw, E.einsum_sq(cw), Pt, 10, out_dtype=torch.int32, with_err=False)
calls = {"lloyd": 0, "iters": 0}
orig = E.lloyd
def lloyd_count(*a, **k):
    C, lab, tr = orig(*a, **k)
    calls["lloyd"] += 1; calls["iters"] += max(len(tr) - 1, 0)  # traces are empty inside DA (labels-only Lloyd)
    return C, lab, tr
E.lloyd = lloyd_count
cfg1 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=1, rel_tol=0.0)
rep = da.TrainReport(config=cfg1)
torch.cuda.synchronize()
_native.prof_enable(True)
t0 = time.perf_counter()
E.da_sweep(X, cw, codes, Pt, sq, cfg1, report=rep)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
_native.prof_enable(False)
prof = _native.prof_collect()
ker = sum(v[1] for v in prof.values()) / 1e3
print(json.dumps({"n": n, "anneal_pass_s": dt, "kernel_s_profiled": ker, "lloyd_calls": calls["lloyd"],
                  "lloyd_iters": calls["iters"], "per_dict_s": [round(s.seconds, 3) for s in rep.steps],
                  "kernels": {k: [v[0], round(v[1], 1)] for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])}}))
