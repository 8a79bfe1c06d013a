"""End-to-end runs of BASELINE.json configs 2 and 3 at full shape on one GPU
(SURVEY §8 row N1 and a9): X_R streamed from pinned host memory as int8
genotype codes (GWG_FORMAT_I8, 1 byte per code), every b_ij streamed out
through a result sink over rotating pinned buffers (c2: 32 GB, c3: 3.2 TB —
never held whole), the order-independent device checksum over every cell,
and seeded random (i, j) spot checks against the oracle (test
infrastructure) and the independent Cholesky route.  Reports e2e GLS/s
against the host-link floor measured on the same box (bare pinned D2H / H2D
copies) and the engine's measured I/O stall.

  python tools/run_configs_e2e.py --config c3 [--m M] [--mb MB] [--ring R]
"""
from __future__ import annotations

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
from oracle import oracle as orc  # noqa: E402
from paper_1210_7683_b200 import datagen  # noqa: E402

SEED = 20261019


def link_bandwidth(nbytes: int = 1 << 30, reps: int = 3) -> dict:
    """Bare pinned copies of nbytes each way (GB/s), CUDA-event timed."""
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[name + "_GBps"] = nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    del h, d
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=["c0", "c1", "c2", "c3", "c4"])
    ap.add_argument("--m", type=int, default=0, help="SNPs (default: the config's m)")
    ap.add_argument("--mb", type=int, default=0)
    ap.add_argument("--ring", type=int, default=3)
    ap.add_argument("--spots", type=int, default=32)
    args = ap.parse_args()
    cfg = datagen.CONFIGS[args.config]
    n, p, t = cfg.n, cfg.p, cfg.t
    m = args.m or cfg.m
    rec = {"config": args.config, "n": n, "p": p, "m": m, "t": t, "cells": m * t,
           "data": "synthetic (BASELINE.json generators, seed %d)" % SEED}
    bw = link_bandwidth()
    rec["link"] = bw

    t0 = time.perf_counter()
    phi = datagen.kinship(SEED, n, cfg.s)
    rec["kinship_build_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    basis, values = gw.eigendecompose(phi, device=0 if n >= 4096 else None)
    rec["eig_s"] = time.perf_counter() - t0
    rec["eig_where"] = "device (cuSOLVER syevd + sign rule)" if n >= 4096 else "CPU LAPACK"
    xl = datagen.covariates(SEED, n, p)
    y_t = torch.empty((t, n), dtype=torch.float64).pin_memory()
    y = y_t.numpy().T
    datagen.normals(SEED, datagen.M_TRAITS, n, 0, t, out=y)
    h2 = datagen.uniform(SEED, datagen.M_H2, t, 0.05, 0.95)
    s2 = np.ones(t)
    t0 = time.perf_counter()
    codes_t = torch.empty((m, n), dtype=torch.int8).pin_memory()
    codes = codes_t.numpy().T  # (n, m) column-major, pinned
    step = max(1, (1 << 28) // (8 * n))
    for a in range(0, m, step):
        k = min(step, m - a)
        codes[:, a:a + k] = datagen.genotypes(SEED, datagen.M_SNPS, n, a, k)
    rec["snp_gen_s"] = time.perf_counter() - t0

    rng = np.random.default_rng(SEED)
    ii = np.sort(rng.integers(0, m, args.spots))
    jj = rng.integers(0, t, args.spots)
    picked = {}
    slabs = [0]

    def sink(i0, cells):
        slabs[0] += 1
        rows = cells.shape[0]
        lo, hi = np.searchsorted(ii, [i0, i0 + rows])
        for k in range(lo, hi):
            picked[k] = cells[ii[k] - i0, jj[k]].copy()

    with gw.Engine(n, p) as eng:
        eng.set_spectrum(basis, values)
        eng.set_covariates(xl)
        eng.set_snp_coding("genotypes")  # int8 codes: the FP64 grid's panels are never read
        eng.reset_counters()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.set_traits(y, h2, s2)
        eng.run_grid(codes, sink=sink, checksum=True, mb=args.mb, ring=args.ring)
        wall = time.perf_counter() - t0
        c = eng.counters()
    h2d = n * m + n * t * 8 + 2 * t * 8
    d2h = m * t * p * 8
    floor = max(h2d / (bw["h2d_GBps"] * 1e9), d2h / (bw["d2h_GBps"] * 1e9))
    rec.update({
        "e2e_s": wall, "e2e_gls_per_s": m * t / wall,
        "h2d_bytes": h2d, "d2h_bytes": d2h,
        "link_floor_s": floor, "e2e_frac_of_link_floor": floor / wall,
        "io_stall_s": c["io_stall_ms"] * 1e-3, "stall_fraction": c["io_stall_ms"] * 1e-3 / wall,
        "grid_kernel_s": c["grid_kernel_ms"] * 1e-3, "rotate_s": c["rotate_ms"] * 1e-3,
        "device_gls_per_s_grid_only": m * t / ((c["grid_kernel_ms"] + c["rotate_ms"]) * 1e-3),
        "checksum": "%#018x" % c["checksum"], "checksum_cells": c["checksum_cells"],
        "slabs": slabs[0], "mb": args.mb or "engine default", "ring": args.ring,
        "api": "Engine.set_traits + Engine.run_grid(int8 codes, sink=..., checksum=True)",
    })
    # spot checks: the oracle's restated compute_tile and the Cholesky route
    got = np.stack([picked[k] for k in range(args.spots)])
    cols, inv_i = np.unique(ii, return_inverse=True)
    tcols, inv_j = np.unique(jj, return_inverse=True)
    workers = os.cpu_count() or 1
    orc.set_blas_threads(workers)
    xs = np.asfortranarray(codes[:, cols].astype(np.float64))
    ref = orc.compute_grid(values, orc.rotate(basis, xl), orc.rotate(basis, xs),
                           orc.rotate(basis, np.asfortranarray(y[:, tcols])), h2[tcols], s2[tcols],
                           workers=workers)
    want = ref[inv_i, inv_j]
    rel = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    fl = np.abs(got - want) / np.maximum(np.abs(want), 1e-5 * np.linalg.norm(want, axis=1,
                                                                             keepdims=True))
    rec["spot_checks"] = {"cells": args.spots, "normwise_max": float(rel.max()),
                          "floored5_componentwise_max": float(fl.max()),
                          "pass": bool(rel.max() <= 1e-10 and fl.max() <= 1e-8)}
    if n <= 2000:
        chol = orc.cholesky_cells(phi, xl, xs, y[:, tcols], h2[tcols], s2[tcols],
                                  inv_i[:8], inv_j[:8])
        crel = np.linalg.norm(got[:8] - chol, axis=1) / np.linalg.norm(chol, axis=1)
        rec["spot_checks"]["cholesky_route_normwise_max"] = float(crel.max())
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
