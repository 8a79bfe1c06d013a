"""PCIe floor of the e2e line on this box: a bare pinned 3.2 GB D2H copy (the
results of one c1 step), and the same with the step's 0.8 GB H2D (the SNP
slab) running concurrently on another stream."""
import time

import torch

x = torch.empty(400_000_000, dtype=torch.float64, device="cuda")
h = torch.empty(400_000_000, dtype=torch.float64).pin_memory()
xs = torch.empty(101_000_000, dtype=torch.float64).pin_memory()
xd = torch.empty(101_000_000, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    h.copy_(x, non_blocking=True)
    torch.cuda.synchronize()


def timed(fn, k=5):
    t = time.perf_counter()
    for _ in range(k):
        fn()
        torch.cuda.synchronize()
    return (time.perf_counter() - t) / k


def both():
    with torch.cuda.stream(s1):
        h.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        xd.copy_(xs, non_blocking=True)


d = timed(lambda: h.copy_(x, non_blocking=True))
u = timed(lambda: xd.copy_(xs, non_blocking=True))
b = timed(both)
print("bare D2H 3.2 GB: %.2f ms (%.1f GB/s); bare H2D 0.81 GB: %.2f ms (%.1f GB/s); "
      "both concurrently: %.2f ms" % (d * 1e3, 3.2 / d, u * 1e3, 0.808 / u, b * 1e3))
