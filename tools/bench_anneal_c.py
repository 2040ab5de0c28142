"""One full anneal pass (da_sweep, 8 dictionaries) on config C (D=960) with a per-kernel breakdown.
usage: python tools/bench_anneal_c.py [n]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E, _native, synthetic

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
X = E.to_dev(np.ascontiguousarray(synthetic.config_c(n=n), dtype=np.float32))
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
t0 = time.perf_counter()
cw, _ = E.growth_pass(X[:50_000].contiguous(), cfg0)
torch.cuda.synchronize()
growth_s = time.perf_counter() - t0
Pt, sq = E.cross_full(cw)
codes, _ = E.encode(X, cw, E.einsum_sq(cw), Pt, 10, out_dtype=torch.int32, with_err=False)
cfg1 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=1, rel_tol=0.0)
out = {"n": n, "D": int(X.shape[1]), "growth_50k_s": round(growth_s, 2)}
for tag, prof in (("pass_s", False), ("pass_profiled_s", True)):
    st = [cw.clone(), codes.clone(), Pt.clone(), sq.clone()]
    rep = da.TrainReport(config=cfg1)
    torch.cuda.synchronize()
    _native.prof_enable(prof)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); E.da_sweep(X, *st, cfg1, report=rep); b.record(); torch.cuda.synchronize()
    _native.prof_enable(False)
    out[tag] = round(a.elapsed_time(b) / 1e3, 3)
    if prof:
        p = _native.prof_collect()
        out["kernels_ms"] = {k: [v[0], round(v[1], 1)] for k, v in sorted(p.items(), key=lambda kv: -kv[1][1])}
    out["distortion_after"] = rep.steps[-1].distortion
print(json.dumps(out))
