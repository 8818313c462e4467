import torch, time
x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
y = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
def t(f, n=10):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n / 1e3
xs = x.view(torch.float32)
print("write-only (fill)  GB/s", (1 << 30) / t(lambda: x.fill_(1)) / 1e9)
print("read-only (sum)    GB/s", (1 << 30) / t(lambda: xs.sum()) / 1e9)
print("copy (r+w bytes)   GB/s", 2 * (1 << 30) / t(lambda: y.copy_(x)) / 1e9)
