"""Development probe: device timeline of the c1 bench step (CUPTI activity
records through torch.profiler): every kernel / memcpy / memset of the last
step with its stream, start offset and duration, so the gaps and the
serialised trait-side work between the three timed launch groups show up.

    python tools/timeline_probe.py [--steps 4] [--option name=value ...]
"""
import argparse
import sys

sys.path.insert(0, ".")
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import os

from paper_1210_7683_b200 import _native as nat

if os.environ.get("TL_LIB"):  # an A/B build (tools/build_variant.sh)
    nat.LIB_PATH = os.environ["TL_LIB"]
import paper_1210_7683_b200 as gw
from paper_1210_7683_b200 import datagen

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--m", type=int, default=100_000)
ap.add_argument("--option", action="append", default=[])
ap.add_argument("--host", action="store_true", help="also list host runtime API calls")
args = ap.parse_args()

n, p, m, t, seed = 1000, 4, args.m, 1000, 20261019
dev = torch.device("cuda", 0)
phi = datagen.kinship(seed, n, 2000)
basis, values = gw.eigendecompose(phi)
xl = datagen.covariates(seed, n, p)
y = torch.from_numpy(np.ascontiguousarray(datagen.normals(seed, datagen.M_TRAITS, n, 0, t).T)).to(dev).t()
h2 = torch.from_numpy(datagen.uniform(seed, datagen.M_H2, t, 0.05, 0.95)).to(dev)
s2 = torch.ones(t, dtype=torch.float64, device=dev)
xh = torch.empty((m, n), dtype=torch.float64).pin_memory()
datagen.genotypes(seed, datagen.M_SNPS, n, 0, m, out=xh.numpy().T)
x = xh.to(dev).t()
b = torch.empty((t, m, p), dtype=torch.float64, device=dev)
eng = gw.Engine(n, p)
eng.set_spectrum(torch.from_numpy(basis).to(dev), torch.from_numpy(values).to(dev))
eng.set_covariates(torch.from_numpy(xl).to(dev))
eng.set_snp_coding("genotypes")
for opt in args.option:
    k, v = opt.split("=", 1)
    eng.set_option(k, int(v))


def step():
    eng.set_traits(y, h2, s2)
    eng.solve_snp_slab(x, out=b, i0=0, layout="stream")


for _ in range(3):
    step()
eng.synchronize()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(args.steps):
        step()
    eng.synchronize()
    torch.cuda.synchronize()

evs = []
for e in prof.events():
    if e.device_type.name == "CUDA" or getattr(e, "device_index", -1) >= 0 and e.is_async:
        pass
for e in prof.profiler.function_events:
    if e.device_type == torch.autograd.DeviceType.CUDA:
        evs.append((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", 0) or e.thread, e.name))
    elif args.host and e.name.startswith("cuda"):
        evs.append((e.time_range.start, e.time_range.end, "H", e.name))
evs.sort()
if not evs:
    print("no device events captured")
    sys.exit(1)
# split into steps at each trait_prep launch (one per set_traits)
starts = [i for i, ev in enumerate(evs) if "trait_prep" in ev[3] and ev[2] != "H"]
print(f"{len(evs)} device events, {len(starts)} steps")
for si in range(len(starts)):
    lo = starts[si]
    hi = starts[si + 1] if si + 1 < len(starts) else len(evs)
    # include events of this step that began before trait_prep (range kernel, Y rotation)
    seg = evs[lo:hi]
    t0 = seg[0][0]
    t_end = max(ev[1] for ev in seg)
    print(f"--- step {si}: span {(t_end - t0) / 1e3:.3f} ms (from trait_prep to the last event)")
    if si == len(starts) - 2 or si == len(starts) - 1:
        busy = 0.0
        last = t0
        for s, e_, strm, name in seg:
            gap = (s - last) / 1e3
            print(f"{(s - t0) / 1e3:8.4f} +{(e_ - s) / 1e3:7.4f} gap {gap:7.4f} s{strm} {name[:90]}")
            last = max(last, e_)
