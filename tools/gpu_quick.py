"""Quick GPU parity probe used during development (not a test)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1210_7683_b200 as gw
from paper_1210_7683_b200 import datagen
from oracle import oracle as orc

for (n, p, m, t) in [(64, 4, 100, 50), (256, 4, 300, 40), (1000, 4, 2000, 100), (200, 1, 50, 9), (300, 7, 130, 21), (500, 20, 70, 13)]:
    ds = datagen.generate(n, p, m, t, seed=11)
    t0 = time.time()
    try:
        res = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"])
    except Exception as e:
        print("ERR", n, p, m, t, type(e).__name__, e); continue
    t1 = time.time()
    ref = orc.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"], workers=8)
    got = res["b"]
    rel = np.linalg.norm(got - ref, axis=2) / np.linalg.norm(ref, axis=2)
    raw = np.abs(got - ref) / np.abs(ref)
    fl = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-6 * np.linalg.norm(ref, axis=2, keepdims=True))
    print(f"n={n} p={p} m={m} t={t}: normwise {rel.max():.3e} raw-comp {raw.max():.3e} floored {fl.max():.3e} nan={np.isnan(got).sum()} gpu {t1-t0:.2f}s counters={res['counters']['kernel_launches']}", flush=True)
