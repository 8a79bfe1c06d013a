"""Seeded synthetic workloads with BASELINE.json's generators.

BASELINE.json names no public dataset; every input is drawn from one seed
(counter-based splitmix64 in csrc/datagen.cpp, so any SNP column range can be
regenerated on its own — by a rank owning a shard, or by a spot check).  The
generator is compiled into the engine library AND into the oracle library
(oracle/Makefile builds the same datagen.cpp), so the CPU reference arm of
bench.py produces bit-identical inputs without loading the engine: every
function takes ``lib=`` (default: the engine library).

* Phi = G G^T / s + 1e-3 I, G n x s standardized Binomial(2, maf) genotypes,
  maf ~ U[0.05, 0.5] per column
* X_L = [1 | N(0,1)^(p-2)]
* X_R  n x m Binomial(2, maf_i) genotypes stored as doubles
* Y    n x t ~ N(0,1);  h2_j ~ U(0.05, 0.95);  sigma2 = 1
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat

M_KINSHIP, M_COVARIATES, M_SNPS, M_TRAITS, M_H2 = 1, 2, 3, 4, 5


@dataclass(frozen=True)
class GridConfig:
    name: str
    n: int
    p: int
    m: int
    t: int
    s: int  # kinship genotype columns


# BASELINE.json "configs" 0..4
CONFIGS = {
    "c0": GridConfig("c0", 1000, 4, 10_000, 100, 2000),
    "c1": GridConfig("c1", 1000, 4, 100_000, 1000, 2000),
    "c2": GridConfig("c2", 10_000, 4, 1_000_000, 1000, 20_000),
    "c3": GridConfig("c3", 1000, 4, 1_000_000, 100_000, 2000),
    "c4": GridConfig("c4", 2000, 20, 200_000, 2000, 2000),
}


def _lib(lib):
    return lib if lib is not None else nat.load()


def genotypes(seed: int, matrix: int, rows: int, col0: int, ncols: int,
              standardize: bool = False, out: np.ndarray | None = None, lib=None) -> np.ndarray:
    lib = _lib(lib)
    if out is None:
        out = np.empty((rows, ncols), dtype=np.float64, order="F")
    assert out.flags.f_contiguous and out.shape == (rows, ncols)
    lib.gwg_gen_genotypes(seed, matrix, rows, col0, ncols, int(standardize),
                          out.ctypes.data, rows)
    return out


def normals(seed: int, matrix: int, rows: int, col0: int, ncols: int,
            out: np.ndarray | None = None, lib=None) -> np.ndarray:
    lib = _lib(lib)
    if out is None:
        out = np.empty((rows, ncols), dtype=np.float64, order="F")
    assert out.flags.f_contiguous and out.shape == (rows, ncols)
    lib.gwg_gen_normals(seed, matrix, rows, col0, ncols, out.ctypes.data, rows)
    return out


def uniform(seed: int, matrix: int, count: int, lo: float, hi: float, lib=None) -> np.ndarray:
    lib = _lib(lib)
    out = np.empty(count, dtype=np.float64)
    lib.gwg_gen_uniform(seed, matrix, count, ctypes.c_double(lo), ctypes.c_double(hi),
                        out.ctypes.data)
    return out


def kinship(seed: int, n: int, s: int, lib=None) -> np.ndarray:
    g = genotypes(seed, M_KINSHIP, n, 0, s, standardize=True, lib=lib)
    phi = (g @ g.T) / float(s)
    phi = 0.5 * (phi + phi.T)
    phi[np.diag_indices(n)] += 1e-3
    return np.asfortranarray(phi)


def covariates(seed: int, n: int, p: int, lib=None) -> np.ndarray:
    xl = np.empty((n, max(p - 1, 0)), dtype=np.float64, order="F")
    if p >= 2:
        xl[:, 0] = 1.0
    if p >= 3:
        normals(seed, M_COVARIATES, n, 0, p - 2, out=xl[:, 1:], lib=lib)
    return xl


def genotype_codes(seed: int, matrix: int, rows: int, col0: int, ncols: int,
                   lib=None) -> np.ndarray:
    """The same genotypes as int8 codes (GWG_FORMAT_I8: 1 byte per code)."""
    out = np.empty((rows, ncols), dtype=np.int8, order="F")
    step = 8192
    for a in range(0, ncols, step):
        k = min(step, ncols - a)
        out[:, a:a + k] = genotypes(seed, matrix, rows, col0 + a, k, lib=lib)
    return out


def generate(n: int, p: int, m: int, t: int, seed: int = 1, s: int | None = None,
             snps_out: np.ndarray | None = None, lib=None) -> dict:
    """A whole dataset as a dict of arrays (the gwgrid.generate shape, with
    BASELINE.json's generators)."""
    s = s if s is not None else 2 * n
    return {
        "kinship": kinship(seed, n, s, lib=lib),
        "xl": covariates(seed, n, p, lib=lib),
        "snps": genotypes(seed, M_SNPS, n, 0, m, out=snps_out, lib=lib),
        "traits": normals(seed, M_TRAITS, n, 0, t, lib=lib),
        "h2": uniform(seed, M_H2, t, 0.05, 0.95, lib=lib),
        "sigma2": np.ones(t, dtype=np.float64),
    }
