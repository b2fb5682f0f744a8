import torch, json
x = torch.empty(1 << 30, dtype=torch.float32, device="cuda")  # 4 GiB
y = torch.empty_like(x)
def t(f, reps=10):
    f(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
    return best
tw = t(lambda: x.fill_(1.0))
tc = t(lambda: y.copy_(x))
tr = t(lambda: x.sum())
n = x.numel() * 4
print(json.dumps({"write_gbs": n / tw / 1e6, "copy_gbs": 2 * n / tc / 1e6, "read_gbs": n / tr / 1e6}))
