"""How much of one dictionary step (heat-up, cool-down, re-encode) of the
config-B anneal pass is GPU-busy time: kernel intervals from the CUDA activity
trace (torch.profiler / CUPTI), merged, against the wall time.  The remainder
is host-bound launch or sync gaps.  usage: python tools/anneal_gaps.py [n]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E
import bench

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n = int(args[0]) if args else 1_000_000
X = E.to_dev(bench.rank_data(0, n))
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(X[:100_000].contiguous(), cfg0)
Pt, sq = E.cross_full(cw)
codes, _ = E.encode(X, cw, E.einsum_sq(cw), Pt, 10, out_dtype=torch.int32, with_err=False)
cfg1 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=1, rel_tol=0.0)
E.dict_step(X, cw.clone(), codes.clone(), Pt.clone(), sq.clone(), 1, cfg1)  # warm-up
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    E.dict_step(X, cw, codes, Pt, sq, 0, cfg1)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
iv = sorted((e.time_range.start, e.time_range.end) for e in prof.events()
            if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start)
busy, cur_s, cur_e, nk = 0.0, None, None, len(iv)
for s, e in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
if cur_e is not None:
    busy += cur_e - cur_s
span = (iv[-1][1] - iv[0][0]) if iv else 0
print(json.dumps({"n": n, "wall_s": wall, "gpu_busy_s": busy / 1e6, "gpu_span_s": span / 1e6, "device_ops": nk,
                  "idle_frac_of_span": 1 - busy / span if span else None}))
if "--table" in sys.argv:
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=60))
