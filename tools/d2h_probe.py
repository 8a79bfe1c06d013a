import torch, time
x = torch.empty(400_000_000, dtype=torch.float64, device="cuda")
h = torch.empty(400_000_000, dtype=torch.float64).pin_memory()
for _ in range(2): h.copy_(x, non_blocking=True); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): h.copy_(x, non_blocking=True); torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print("bare D2H 3.2 GB: %.2f ms, %.1f GB/s" % (dt * 1e3, 3.2 / dt))
