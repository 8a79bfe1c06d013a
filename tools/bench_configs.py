"""Device throughput on every BASELINE.json config (informational; bench.py is
the contract line).  Full n, p, t; a representative SNP slab resident in HBM
(the grid is a sum of independent slabs).  Prints one JSON line per config.

  python tools/bench_configs.py [--configs c0,c1,c2,c3,c4] [--steps 3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1210_7683_b200 as gw  # noqa: E402
from paper_1210_7683_b200 import datagen  # noqa: E402

PEAK = 37.15
SLAB = {"c0": 10_000, "c1": 100_000, "c2": 100_000, "c3": 4_736, "c4": 50_000,
        "p8": 50_000, "p12": 50_000, "p13": 50_000, "n2k": 50_000, "n4k": 50_000,
        "n6k": 50_000}
EXTRA = {"p8": datagen.GridConfig("p8", 1000, 8, 50_000, 1000, 2000),
         "p12": datagen.GridConfig("p12", 1000, 12, 50_000, 1000, 2000),
         "p13": datagen.GridConfig("p13", 1000, 13, 50_000, 1000, 2000),
         "n2k": datagen.GridConfig("n2k", 2000, 4, 50_000, 1000, 4000),
         "n4k": datagen.GridConfig("n4k", 4000, 4, 50_000, 1000, 8000),
         "n6k": datagen.GridConfig("n6k", 6000, 4, 50_000, 1000, 12000)}


def run(name, steps, options=()):
    cfg = datagen.CONFIGS.get(name) or EXTRA[name]
    n, p, t, m = cfg.n, cfg.p, cfg.t, SLAB[name]
    seed = 7
    dev = torch.device("cuda", 0)
    t0 = time.perf_counter()
    phi = datagen.kinship(seed, n, cfg.s)
    t1 = time.perf_counter()
    basis, values = gw.eigendecompose(phi, device=0)
    t2 = time.perf_counter()
    xl = datagen.covariates(seed, n, p)
    y = torch.from_numpy(np.ascontiguousarray(datagen.normals(seed, datagen.M_TRAITS, n, 0, t).T)).to(dev).t()
    h2 = torch.from_numpy(datagen.uniform(seed, datagen.M_H2, t, 0.05, 0.95)).to(dev)
    s2 = torch.ones(t, dtype=torch.float64, device=dev)
    xh = torch.empty((m, n), dtype=torch.float64)
    datagen.genotypes(seed, datagen.M_SNPS, n, 0, m, out=xh.numpy().T)
    x = xh.to(dev).t()
    b = torch.empty((m, t, p), dtype=torch.float64, device=dev)
    with gw.Engine(n, p) as eng:
        eng.set_spectrum(basis, values)
        eng.set_covariates(xl)
        eng.set_snp_coding(os.environ.get("GWG_SNP_CODING", "genotypes"))
        for opt in options:
            k, v = opt.split("=")
            eng.set_option(k, int(v))
        stream = torch.cuda.ExternalStream(eng.compute_stream, device=dev)

        def step():
            eng.set_traits(y, h2, s2)
            eng.solve_snp_slab(x, out=b)

        step()
        torch.cuda.synchronize()
        eng.reset_counters()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            step()
        eng.synchronize()  # device-output solves are asynchronous: read their error words
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        c = eng.counters()
    kern = c["grid_kernel_ms"] / steps
    grid_flops = m * t * 2 * n * (p + 1)
    return {"build": os.environ.get("GWG_BUILD_TAG", ""), "options": list(options), "config": name, "n": n, "p": p, "t": t, "m_slab": m, "ms_per_step": ms,
            "gls_per_s": m * t / (ms * 1e-3), "step_tflops_grid_convention": grid_flops / ms / 1e9,
            "grid_kernel_ms": kern, "grid_kernel_tflops": grid_flops / kern / 1e9,
            "grid_kernel_frac_of_peak": grid_flops / kern / 1e9 / PEAK,
            "rotate_ms": c["rotate_ms"] / steps, "sbr_ms": c["quad_ms"] / steps,
            "linear_solve_ms": c["linear_ms"] / steps, "sbr_terms": c["sbr_terms"],
            "kinship_build_s": t1 - t0,
            "device_eig_s": t2 - t1, "nan": int(torch.isnan(b).sum().item())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c0,c1,c2,c3,c4")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--option", action="append", default=[], metavar="NAME=VALUE",
                    help="engine option (gwg_set_option), e.g. i8_cluster=4")
    args = ap.parse_args()
    for name in args.configs.split(","):
        print(json.dumps(run(name, args.steps, args.option)), flush=True)


if __name__ == "__main__":
    main()
