"""Config C (D=960) encode rates on a 200k-vector subsample (synthetic mixture)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E, synthetic, _native
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
X_h = synthetic.config_c(n=n) if "n" in synthetic.config_c.__code__.co_varnames else synthetic.config_c(n)
X = E.to_dev(np.ascontiguousarray(X_h, dtype=np.float32))
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
t0 = time.perf_counter()
cw, _ = E.growth_pass(X[:50000].contiguous(), cfg0)
torch.cuda.synchronize()
out = {"n": n, "D": X.shape[1], "growth_50k_s": time.perf_counter() - t0}
Pt, _ = E.cross_full(cw); sq = E.einsum_sq(cw)
for L in (1, 10):
    E.encode(X, cw, sq, Pt, L, out_dtype=torch.uint8, with_err=False); torch.cuda.synchronize()
    t0 = time.perf_counter(); E.encode(X, cw, sq, Pt, L, out_dtype=torch.uint8, with_err=False); torch.cuda.synchronize()
    out[f"L={L} vectors/s"] = n / (time.perf_counter() - t0)
    rc = torch.zeros(1, dtype=torch.int64, device="cuda")
    E.encode_config(0, rc)
    _native.prof_enable(True)
    codes_L = E.encode(X, cw, sq, Pt, L, out_dtype=torch.uint8, with_err=False)[0]; torch.cuda.synchronize()
    _native.prof_enable(False)
    E.encode_config(0)
    M, K = cw.shape[0], cw.shape[1]
    out[f"L={L} recheck_fraction"] = float(rc.item()) / (n * sum(min(L, K ** m) * K for m in range(M)))
    out[f"L={L} codes_sha"] = __import__("hashlib").sha256(codes_L.cpu().numpy().tobytes()).hexdigest()[:16]
    out[f"L={L} kernels_ms"] = {k: round(v[1], 3) for k, v in _native.prof_collect().items()}
print(json.dumps(out))
