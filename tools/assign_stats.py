"""Exact rechecks per row in the tcgen05 assign (bench_assign data)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_05194_b200 import _engine as E
import bench
n = 1_000_000
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((n, 128), dtype=torch.float64, device="cuda", generator=g) * 30
C = X[torch.randint(0, n, (256,), device="cuda", generator=g)] + torch.randn((256, 128), dtype=torch.float64, device="cuda", generator=g)
Xb = E.to_dev(bench.rank_data(0, n)).double()
Cb = Xb[torch.randint(0, n, (256,), device="cuda", generator=g)].contiguous()
for name, XX, CC in (("random", X, C), ("configB", Xb, Cb)):
    for d in (8, 32, 128):
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        E.assign_config(0, cnt)
        E.assign(XX, d, CC)
        torch.cuda.synchronize()
        print(name, d, "rechecks/row", cnt.item() / n, flush=True)
E.assign_config(0)
