import torch, time
x = torch.empty(1280000000 // 8, dtype=torch.float64).pin_memory()
y = torch.empty_like(x, device="cuda")
o = torch.empty(490837644 // 8, dtype=torch.float64, device="cuda")
ob = torch.empty_like(o, device="cpu").pin_memory()
for _ in range(2): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"H2D 1.28 GB: {dt*1e3:.2f} ms = {1.28/dt:.1f} GB/s")
s2 = torch.cuda.Stream()
t = time.perf_counter()
for _ in range(5):
    y.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        ob.copy_(o, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"H2D 1.28 GB + concurrent D2H 0.49 GB: {dt*1e3:.2f} ms")
