"""Small end-to-end case for compute-sanitizer runs (one tool per gpurun call).

  python tools/sanitize_case.py [real|genotypes]
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1210_7683_b200 as gw  # noqa: E402
from paper_1210_7683_b200 import datagen  # noqa: E402

coding = sys.argv[1] if len(sys.argv) > 1 else "real"
for (n, p, m, t) in ((130, 4, 150, 37), (96, 1, 40, 9), (200, 8, 70, 20), (64, 20, 30, 9),
                     (300, 3, 260, 70)):
    ds = datagen.generate(n, p, m, t, seed=3)
    z, lam = gw.eigendecompose(ds["kinship"])
    with gw.Engine(n, p) as eng:
        eng.set_spectrum(z, lam)
        eng.set_covariates(ds["xl"])
        eng.set_snp_coding(coding)
        eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
        b = eng.run_grid(ds["snps"], mb=64)
        b2 = eng.solve_snp_slab(ds["snps"])
        bs = eng.run_grid(ds["snps"], layout="stream", mb=100)
        assert np.array_equal(b, b2) and not np.isnan(b).any()
        assert np.array_equal(bs.transpose(1, 0, 2), b)
    err = gw.verify_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                         ds["sigma2"], b)
    print(n, p, m, t, "verify", err)
z2, l2 = gw.eigendecompose(datagen.kinship(1, 300, 600), device=0)
print("ok")

# round-2 paths: int8 input, sinks, checksum, asynchronous device solves in
# both layouts, the device group
import torch  # noqa: E402

ds = datagen.generate(200, 4, 300, 40, seed=9)
z, lam = gw.eigendecompose(ds["kinship"])
codes = ds["snps"].astype(np.int8)
with gw.Engine(200, 4) as eng:
    eng.set_spectrum(z, lam)
    eng.set_covariates(ds["xl"])
    eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
    b = eng.run_grid(codes, checksum=True, mb=70)
    got = np.empty_like(b)

    def sink(i0, cells):
        got[i0:i0 + cells.shape[0]] = cells

    eng.run_grid(ds["snps"], sink=sink, mb=64, ring=3)
    assert np.array_equal(got, b)
    x = torch.from_numpy(ds["snps"]).cuda()
    out = torch.empty((300, 40, 4), dtype=torch.float64, device="cuda")
    outs = torch.empty((40, 300, 4), dtype=torch.float64, device="cuda")
    eng.solve_snp_slab(x, out=out)
    eng.solve_snp_slab(x, out=outs, layout="stream")
    eng.synchronize()
    assert np.array_equal(out.cpu().numpy(), b)
    assert np.array_equal(outs.cpu().numpy().transpose(1, 0, 2), b)
with gw.Group(200, 4, [0, 0]) as g:
    g.set_spectrum(z, lam)
    g.set_covariates(ds["xl"])
    g.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
    assert np.array_equal(g.run_grid(codes, mb=50), b)
print("round-2 paths ok")
