import torch, time
x = torch.empty(2*1024**3, dtype=torch.float32, device="cuda")  # 8 GB
y = torch.empty_like(x)
def t(f, n=5):
    f(); torch.cuda.synchronize()
    a,b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)/n
ms = t(lambda: x.fill_(1.0)); print("fill 8GB: %.2f ms = %.2f TB/s write" % (ms, 8.59/ms))
ms = t(lambda: x.sum()); print("sum 8GB: %.2f ms = %.2f TB/s read" % (ms, 8.59/ms))
ms = t(lambda: y.copy_(x)); print("copy 8GB: %.2f ms = %.2f TB/s r+w" % (ms, 2*8.59/ms))
