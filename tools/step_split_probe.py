"""Development probe: the c1 bench step split into gwg_set_traits and
gwg_solve_snp_slab, each timed alone with CUDA events on the engine stream."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1210_7683_b200 as gw
from paper_1210_7683_b200 import datagen

n, p, m, t, seed = 1000, 4, 100_000, 1000, 20261019
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
b = torch.empty((m, t, p), dtype=torch.float64, device=dev)
eng = gw.Engine(n, p)
eng.set_spectrum(torch.from_numpy(basis).to(dev), torch.from_numpy(values).to(dev))
eng.set_covariates(torch.from_numpy(xl).to(dev))
eng.set_snp_coding("genotypes")
st = torch.cuda.ExternalStream(eng.compute_stream, device=dev)


def timed(fn, k=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(k):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


both = timed(lambda: (eng.set_traits(y, h2, s2), eng.solve_snp_slab(x, out=b)))
tr = timed(lambda: eng.set_traits(y, h2, s2))
eng.set_traits(y, h2, s2)
eng.solve_snp_slab(x, out=b)
sl = timed(lambda: eng.solve_snp_slab(x, out=b))
print(f"step {both:.3f} ms = set_traits alone {tr:.3f} + solve alone {sl:.3f} (sum {tr + sl:.3f})")
