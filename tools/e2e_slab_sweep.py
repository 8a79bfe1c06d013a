"""c1 end to end (set_traits + run_grid from pinned host buffers) over slab widths and both input
formats: measured flat on the B200 (f64 63.8-64.9 ms for mb 1,024..8,192, int8 62.4-63.4 ms;
bare 3.2 GB D2H on the same box 58.3 ms), i.e. the e2e step is the result transfer plus a
fixed ~1.6 ms head, not a slab-size effect.  Run under gpurun."""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1210_7683_b200 as gw
from paper_1210_7683_b200 import datagen
n,p,m,t=1000,4,100000,1000
ds = datagen.generate(n,p,2000,t,seed=3)
basis, values = gw.eigendecompose(ds["kinship"])
x = torch.empty((m,n), dtype=torch.float64).pin_memory()
datagen.genotypes(3, datagen.M_SNPS, n, 0, m, out=x.numpy().T)
xi8 = torch.empty((m,n), dtype=torch.int8).pin_memory(); xi8.copy_(x.to(torch.int8))
b = torch.empty((m,t,p), dtype=torch.float64).pin_memory()
with gw.Engine(n,p) as eng:
    eng.set_spectrum(basis, values); eng.set_covariates(ds["xl"]); eng.set_snp_coding("genotypes")
    for name, src in (("f64", x.numpy().T), ("i8", xi8.numpy().T)):
        for mb in (0, 1024, 2048, 4096, 8192, 16384, 32768):
            ts=[]
            for r in range(4):
                torch.cuda.synchronize(); t0=time.perf_counter()
                eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
                eng.run_grid(src, out=b.numpy(), layout="numpy", mb=mb)
                ts.append(time.perf_counter()-t0)
            print(name, "mb", mb, "ms", [round(v*1e3,2) for v in ts], "stall", round(eng.counters()["io_stall_ms"],1), flush=True)
