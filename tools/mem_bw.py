import torch, json
x = torch.empty(1 << 29, dtype=torch.float32, device="cuda")  # 2 GiB
y = torch.empty_like(x)
def t(f, n=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
b = x.numel() * 4
print(json.dumps({"fill_GBps": round(b / t(lambda: x.fill_(1.0)) / 1e6, 1),
                  "copy_GBps_rw": round(2 * b / t(lambda: y.copy_(x)) / 1e6, 1),
                  "read_sum_GBps": round(b / t(lambda: x.sum()) / 1e6, 1)}))
