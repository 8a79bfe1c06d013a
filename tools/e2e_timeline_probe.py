"""Development probe: device timeline of the c1 e2e step (gwg_set_traits +
gwg_run_grid from pinned host buffers, X_R as float64): per stream, the busy
time of copies and kernels and the idle gaps of the D2H stream, to find what
separates the step from the PCIe floor.

    python tools/e2e_timeline_probe.py [--mb MB] [--i8]
"""
import argparse
import sys

sys.path.insert(0, ".")
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1210_7683_b200 as gw
from paper_1210_7683_b200 import datagen

ap = argparse.ArgumentParser()
ap.add_argument("--mb", type=int, default=0)
ap.add_argument("--i8", action="store_true")
args = ap.parse_args()
n, p, m, t, seed = 1000, 4, 100_000, 1000, 20261019
phi = datagen.kinship(seed, n, 2000)
basis, values = gw.eigendecompose(phi)
xl = datagen.covariates(seed, n, p)
y = np.asfortranarray(datagen.normals(seed, datagen.M_TRAITS, n, 0, t))
h2 = datagen.uniform(seed, datagen.M_H2, t, 0.05, 0.95)
s2 = np.ones(t)
xh_t = torch.empty((m, n), dtype=torch.float64).pin_memory()
datagen.genotypes(seed, datagen.M_SNPS, n, 0, m, out=xh_t.numpy().T)
x = xh_t.numpy().T
if args.i8:
    x8_t = torch.empty((m, n), dtype=torch.int8).pin_memory()
    x8_t.copy_(xh_t.to(torch.int8))
    x = x8_t.numpy().T
b_t = torch.empty((m, t, p), dtype=torch.float64).pin_memory()
b = b_t.numpy()
eng = gw.Engine(n, p)
eng.set_spectrum(basis, values)
eng.set_covariates(xl)
eng.set_snp_coding("genotypes")


def step():
    eng.set_traits(y, h2, s2)
    eng.run_grid(x, out=b, layout="numpy", mb=args.mb)


for _ in range(2):
    step()
torch.cuda.synchronize()
import time as _t
for _ in range(3):
    a = _t.perf_counter()
    eng.set_traits(y, h2, s2)
    b_ = _t.perf_counter()
    eng.run_grid(x, out=b, layout="numpy", mb=args.mb)
    c = _t.perf_counter()
    print(f"host: set_traits {1e3 * (b_ - a):.3f} ms, run_grid {1e3 * (c - b_):.3f} ms")
import time
t0 = time.perf_counter()
step()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
evs = []
for e in prof.profiler.function_events:
    if e.device_type == torch.autograd.DeviceType.CUDA:
        evs.append((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", 0) or e.thread, e.name))
evs.sort()
t0 = evs[0][0]
span = (max(e[1] for e in evs) - t0) / 1e3
print(f"wall {wall:.2f} ms (unprofiled), profiled device span {span:.2f} ms, {len(evs)} events")
streams = {}
for s, e_, st, name in evs:
    streams.setdefault(st, []).append((s, e_, name))
for st, lst in streams.items():
    busy = sum(e_ - s for s, e_, _ in lst) / 1e3
    kinds = {}
    for s, e_, name in lst:
        k = "D2H" if "DtoH" in name else "H2D" if "HtoD" in name else name.split("(")[0][-40:]
        kinds[k] = kinds.get(k, 0.0) + (e_ - s) / 1e3
    first, last = (lst[0][0] - t0) / 1e3, (lst[-1][1] - t0) / 1e3
    print(f"stream {st}: {len(lst)} events, busy {busy:.2f} ms in [{first:.2f}, {last:.2f}]; " +
          ", ".join(f"{k} {v:.2f}" for k, v in sorted(kinds.items(), key=lambda kv: -kv[1])[:6]))
    d2h = [(s, e_) for s, e_, name in lst if "DtoH" in name]
    if len(d2h) > 3:
        gaps = [(d2h[i + 1][0] - d2h[i][1]) / 1e3 for i in range(len(d2h) - 1)]
        durs = [(e_ - s) / 1e3 for s, e_ in d2h]
        print(f"   D2H: {len(d2h)} copies, mean {np.mean(durs):.3f} ms (max {max(durs):.3f}), "
              f"gaps total {sum(gaps):.2f} ms (max {max(gaps):.3f})")
