"""Development probe (not a test): the cta_group::2 int8 path (GWG_I8_CLUSTER=3)
against the multicast path, bit for bit, then c1-size timings of both."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ".")
    import numpy as np
    import paper_1210_7683_b200 as gw
    from paper_1210_7683_b200 import datagen
    out = {}
    for (n, p, m, t) in [(200, 4, 300, 20), (1000, 4, 1000, 64), (257, 20, 333, 7), (300, 12, 129, 17)]:
        ds = datagen.generate(n, p, m, t, seed=n + p)
        basis, values = gw.eigendecompose(ds["kinship"])
        with gw.Engine(n, p) as eng:
            eng.set_spectrum(basis, values)
            eng.set_covariates(ds["xl"])
            eng.set_snp_coding("genotypes")
            eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
            b = eng.run_grid(ds["snps"])
        np.save("gpurun_out/pc_%s_%d_%d.npy" % (os.environ["GWG_I8_CLUSTER"], n, p), b)
        print(os.environ["GWG_I8_CLUSTER"], n, p, "nan", int(np.isnan(b).sum()), flush=True)
    sys.exit(0)

import numpy as np
for cl in ("2", "3", "4"):
    env = dict(os.environ, GWG_I8_CLUSTER=cl)
    r = subprocess.run(["timeout", "120", sys.executable, __file__, "child"], env=env)
    print("cl", cl, "rc", r.returncode, flush=True)
    if r.returncode != 0:
        sys.exit(1)
for (n, p) in [(200, 4), (1000, 4), (257, 20), (300, 12)]:
    a = np.load("gpurun_out/pc_2_%d_%d.npy" % (n, p))
    for cl in ("3", "4"):
        b = np.load("gpurun_out/pc_%s_%d_%d.npy" % (cl, n, p))
        print(cl, n, p, "bitwise equal" if np.array_equal(a, b) else "DIFF max %g" % np.nanmax(np.abs(a - b)))
