"""Print a hash of the device grid for one engine build (bitwise A/B of two
builds that must agree bit for bit):
  python tools/lib_bits.py tools/_exp/libA.so [n p m t]
"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1210_7683_b200 import _native as nat

nat.LIB_PATH = sys.argv[1]
import paper_1210_7683_b200 as gw  # noqa: E402
from paper_1210_7683_b200 import datagen  # noqa: E402

n, p, m, t = (int(v) for v in (sys.argv[2:6] if len(sys.argv) >= 6 else (1000, 4, 20000, 300)))
ds = datagen.generate(n, p, m, t, seed=5)
basis, values = gw.eigendecompose(ds["kinship"], device=0 if n >= 4096 else None)
out = []
for coding in ("genotypes", "real"):
    with gw.Engine(n, p) as eng:
        eng.set_spectrum(basis, values)
        eng.set_covariates(ds["xl"])
        eng.set_snp_coding(coding)
        eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
        b = eng.run_grid(ds["snps"])
    out.append("%s %s nan=%d" % (coding, hashlib.sha256(np.ascontiguousarray(b).tobytes()).hexdigest()[:16],
                                 int(np.isnan(b).sum())))
print(sys.argv[1].split("/")[-1], n, p, m, t, " | ".join(out))
