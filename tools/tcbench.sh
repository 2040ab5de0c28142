timeout 300 python tools/debug_tc_b.py 2>&1 | tail -3
DA_DEBUG=1 timeout 120 python tools/prof_tc.py 3 10 2>&1 | grep encode_tc | head -2
timeout 300 python -m pytest tests/test_gpu_encode_paths.py -m gpu -q -x > gpurun_out/p.log 2>&1; tail -1 gpurun_out/p.log
python -c "
import sys, os, torch, time; sys.path.insert(0, \".\")
import bench
from paper_1509_05194_b200 import _engine as E
import paper_1509_05194_b200 as da
X = E.to_dev(bench.rank_data(0, 1000000)); cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(X[:100000].contiguous(), cfg0); Pt, sq = E.cross_full(cw); sqe = E.einsum_sq(cw)
for mode in (2, 3):
  for L in (1, 10):
    E.encode_config(mode); E.encode(X, cw, sqe, Pt, L, with_err=False); torch.cuda.synchronize()
    t0 = time.perf_counter(); E.encode(X, cw, sqe, Pt, L, with_err=False); torch.cuda.synchronize(); print(mode, L, round(time.perf_counter() - t0, 4))
"
