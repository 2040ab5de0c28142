"""Where the end-to-end encode time goes (host copies, pinned alloc, upload, encode)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_05194_b200 as da
from paper_1509_05194_b200 import _engine as E
import bench
n = 1000000
X = bench.rank_data(0, n)
Xd = E.to_dev(X)
cfg0 = da.TrainConfig(m_count=8, k_count=256, beam_width=10, sweeps=0, rel_tol=0.0)
cw, _ = E.growth_pass(Xd[:100000].contiguous(), cfg0)
Pt, _ = E.cross_full(cw); sq = E.einsum_sq(cw)
torch.cuda.synchronize()
def t(f, label, rep=2):
    best = 1e9
    for _ in range(rep):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    print(f"{label:40s} {best*1e3:8.1f} ms", flush=True)
t(lambda: torch.empty((131072, 128), dtype=torch.float32, pin_memory=True), "pinned alloc 64MB")
pin = torch.empty((n, 128), dtype=torch.float32, pin_memory=True)
t(lambda: np.copyto(pin.numpy(), X), "np.copyto 512MB -> pinned")
t(lambda: Xd.copy_(pin, non_blocking=True), "H2D 512MB from pinned")
t(lambda: torch.from_numpy(X).to("cuda"), "pageable H2D 512MB")
t(lambda: np.isfinite(X).all(), "np.isfinite 512MB")
t(lambda: E.encode(Xd, cw, sq, Pt, 10, out_dtype=torch.uint8, with_err=False), "device encode L=10")
t(lambda: E.encode_host(X, cw, sq, Pt, 10, out_dtype=torch.uint8), "encode_host L=10")
t(lambda: E.encode_host(X, cw, sq, Pt, 10, out_dtype=torch.uint8, chunk=262144), "encode_host L=10 chunk 256K")
