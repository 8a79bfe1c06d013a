"""Golden b vectors written by the REFERENCE itself (TEST INFRASTRUCTURE).

`python -m tests.golden.make_ref_golden` runs the reference's own sources —
compiled where they lie under /root/reference into oracle/_ref/ by
oracle/refbuild/Makefile (against our Eigen stand-in; see oracle/ref.py) —
through its gwgrid.solve_grid route (python/bindings.cpp:115-190: GWG1 files,
preloop_stream_transform, run_grid CT) on seeded inputs from BASELINE.json's
generators, and stores the resulting grids in tests/golden/ref_grids.npz with
the reference's dense-Cholesky route (CholeskyOracle, gls.cpp:188-244) at a
few cells.  Only the seeds and the outputs are stored: the inputs regenerate
bit-identically from the counter-based generator (engine library on the GPU
box, the oracle library's copy of it in the CPU tests).

/root/reference does not exist on the GPU box, so the GPU tests read the
committed file; tests/test_ref_pin.py re-runs the reference here and checks
that the committed vectors are what it produces.
"""
from __future__ import annotations

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATH = os.path.join(HERE, "ref_grids.npz")

# name: (n, p, m, t, seed, SNP kind).  "codes" = BASELINE's genotype codes
# {0,1,2}; "real" = standard normals (the all-FP64 device path).  t >= 256
# exercises the device's factorised S_BR / W build, p = 1 the no-covariate
# cell, p = 20 config 4's width, n = 1000 configs 0/1/3's.
CASES = {
    "codes_n64_p4": (64, 4, 50, 30, 3, "codes"),
    "codes_n100_p1": (100, 1, 40, 20, 5, "codes"),
    "codes_n128_p7": (128, 7, 33, 17, 6, "codes"),
    "codes_n200_p20": (200, 20, 24, 12, 8, "codes"),
    "codes_n300_p4_t256": (300, 4, 36, 256, 9, "codes"),
    "codes_n1000_p4": (1000, 4, 128, 64, 20260816, "codes"),
    "real_n96_p3": (96, 3, 40, 24, 4, "real"),
    "real_n1000_p4": (1000, 4, 48, 32, 12, "real"),
}
N_CHOLESKY_CELLS = 6


def inputs(name: str, lib=None) -> dict:
    """The case's operands from the counter-based generator in `lib` (the
    engine library by default; pass oracle.load() to stay off the engine)."""
    from paper_1210_7683_b200 import datagen

    n, p, m, t, seed, kind = CASES[name]
    ds = datagen.generate(n, p, m, t, seed=seed, lib=lib)
    if kind == "real":
        ds["snps"] = datagen.normals(seed, datagen.M_SNPS, n, 0, m, lib=lib)
    return ds


def cholesky_cells(name: str):
    n, p, m, t, seed, _ = CASES[name]
    rng = np.random.default_rng(seed + 1000)
    return rng.integers(0, m, N_CHOLESKY_CELLS), rng.integers(0, t, N_CHOLESKY_CELLS)


def run_reference(name: str, lib=None) -> dict:
    from oracle import ref

    ds = inputs(name, lib=lib)
    b = ref.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"],
                       scheduler="ct", workers=2)
    ci, cj = cholesky_cells(name)
    chol = ref.cholesky_cells(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                              ds["sigma2"], ci, cj)
    return {"b": b, "chol": chol}


def load() -> dict:
    with np.load(PATH) as z:
        return {name: {"b": z[name + "/b"], "chol": z[name + "/chol"]} for name in CASES}


def main() -> None:
    from oracle import oracle as orc

    out = {}
    for name in CASES:
        got = run_reference(name, lib=orc.load())
        out[name + "/b"] = got["b"]
        out[name + "/chol"] = got["chol"]
        print(name, got["b"].shape, f"{got['b'].nbytes / 1024:.0f} KiB")
    np.savez(PATH, **out)
    print("wrote", PATH, f"{os.path.getsize(PATH) / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
