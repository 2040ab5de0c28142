import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_05194_b200 import _engine as E
n, K = 1_000_000, 256
D = int(sys.argv[1]) if len(sys.argv) > 1 else 128
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((n, 128), dtype=torch.float64, device="cuda", generator=g)
lab = torch.randint(0, K, (n,), dtype=torch.int32, device="cuda", generator=g)
C = torch.zeros((K, 128), dtype=torch.float64, device="cuda")
cnt = torch.zeros(K, dtype=torch.int32, device="cuda")
def run():
    E.native.da_group_sums(E.P(X), n, 128, D, E.P(lab), K, 0, E.P(C), 128, E.P(cnt), E.stream())
for _ in range(3): run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): run()
e1.record(); torch.cuda.synchronize()
print(json.dumps({"group_sums_ms": e0.elapsed_time(e1) / 10}))
