import torch, time
x = torch.empty(128 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty_like(x, device="cuda")
for sz in (8 << 20, 32 << 20, 128 << 20):
    ts = []
    for _ in range(10):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        d[:sz].copy_(x[:sz], non_blocking=True); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print("H2D", sz >> 20, "MB", round(sz / min(ts) / 1e9, 1), "GB/s")
# concurrent H2D + D2H
y = torch.empty(128 << 20, dtype=torch.uint8).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(x, non_blocking=True)
with torch.cuda.stream(s2): y.copy_(d, non_blocking=True)
torch.cuda.synchronize(); print("duplex", round(2 * (128 << 20) / (time.perf_counter() - t0) / 1e9, 1), "GB/s")
