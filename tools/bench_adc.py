"""ADC candidate-list scan (config E shape): nq queries x ncand random candidate ids
over N encoded vectors; per-query top-r.  Times the scan kernel with CUDA events."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_05194_b200 import _engine as E
N = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000
ncand = int(sys.argv[3]) if len(sys.argv) > 3 else 100_000
M, K, D, r = 8, 256, 128, 100
g = torch.Generator(device="cuda").manual_seed(4)
codes = torch.randint(0, K, (N, M), dtype=torch.uint8, device="cuda", generator=g)
pair = torch.rand(N, dtype=torch.float64, device="cuda", generator=g)
cw = torch.randn((M, K, D), dtype=torch.float32, device="cuda", generator=g)
sq = E.einsum_sq(cw)
Q = torch.randn((nq, D), dtype=torch.float64, device="cuda", generator=g)
lut, qsq = E.adc_lut(Q, cw, sq)
cand = torch.randint(0, N, (nq, ncand), dtype=torch.int64, device="cuda", generator=g)
E.adc_scan(codes, pair, lut[:16], qsq[:16], r, cand=cand[:16])
torch.cuda.synchronize()
rec = E.adc_pack(codes, pair)
for name, fn in (("generic", lambda: E.adc_scan(codes, pair, lut, qsq, r, cand=cand)),
                 ("packed", lambda: E.adc_scan_packed(rec, lut, qsq, r, cand=cand))):
    fn()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    ids, d = fn()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    tot = nq * ncand
    print(f"{name}: N={N} nq={nq} ncand={ncand}: {ms:.2f} ms, {tot / ms / 1e6:.1f} G cand/s, "
          f"{40 * tot / ms / 1e6:.0f} GB/s at 40 B/cand (algorithmic)", flush=True)
