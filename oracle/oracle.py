"""ctypes face of oracle/gls_oracle.cpp — TEST INFRASTRUCTURE ONLY.

The CPU restatement of the reference gwgrid hot path (see the header of
gls_oracle.cpp for the file:line map).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this module;
the product package never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libgls_oracle.so")


class OracleError(Exception):
    def __init__(self, code: int, msg: str, snp_index: int, trait_index: int):
        super().__init__(msg)
        self.code = code
        self.snp_index = snp_index
        self.trait_index = trait_index


class _Status(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("snp_index", ctypes.c_int64),
                ("trait_index", ctypes.c_int64), ("msg", ctypes.c_char * 256)]


CODES = {1: "dimension", 2: "non_symmetric", 3: "backend", 4: "not_positive_definite"}

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB_PATH


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        lib = ctypes.CDLL(LIB_PATH)
        P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        S = ctypes.POINTER(_Status)
        for name, args in {
            "orc_eigendecompose": [I64, P, P, P, S],
            "orc_rotate": [I64, P, I64, P, P],
            "orc_trait_weights": [I64, P, D, D, I64, P, P, S],
            "orc_trait_context": [I64, I64, P, P, P, D, D, I64, P, P, P, P, S],
            "orc_solve_partitioned": [I64, I64, P, P, P, P, P, D, D, P, S],
            "orc_solve_single": [I64, I64, P, P, P, P, D, D, P, S],
            "orc_cholesky_solve": [I64, I64, P, P, P, D, D, P, S],
            "orc_cholesky_cells": [I64, I64, I64, I64, P, P, P, P, P, P, I64, P, P, P, S],
            "orc_compute_grid": [I64, I64, I64, I64, P, P, P, P, P, P, I64, I64, I32, I32, P, S],
            "orc_solve_grid": [I64, I64, I64, I64, P, P, P, P, P, P, I32, I32, P, S],
        }.items():
            fn = getattr(lib, name)
            fn.restype = ctypes.c_int32
            fn.argtypes = args
        U64, PD = ctypes.c_uint64, ctypes.c_void_p
        lib.gwg_gen_genotypes.argtypes = [U64, I32, I64, I64, I64, I32, PD, I64]
        lib.gwg_gen_genotypes.restype = None
        lib.gwg_gen_normals.argtypes = [U64, I32, I64, I64, I64, PD, I64]
        lib.gwg_gen_normals.restype = None
        lib.gwg_gen_uniform.argtypes = [U64, I32, I64, D, D, PD]
        lib.gwg_gen_uniform.restype = None
        lib.orc_set_blas_threads.argtypes = [ctypes.c_int]
        lib.orc_set_blas_threads.restype = None
        lib.orc_cell_flops.restype = ctypes.c_uint64
        lib.orc_cell_flops.argtypes = [I64, I64]
        _lib = lib
    return _lib


def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _check(rc: int, st: _Status) -> None:
    if rc != 0:
        raise OracleError(rc, st.msg.decode(errors="replace"), st.snp_index, st.trait_index)


def set_blas_threads(n: int) -> None:
    load().orc_set_blas_threads(int(n))


def eigendecompose(phi):
    phi = _f(phi)
    n = phi.shape[0]
    basis = np.empty((n, n), order="F")
    values = np.empty(n)
    st = _Status()
    _check(load().orc_eigendecompose(n, _ptr(phi), _ptr(basis), _ptr(values), ctypes.byref(st)), st)
    return basis, values


def rotate(basis, src):
    basis, src = _f(basis), _f(src)
    if src.ndim == 1:
        src = src.reshape(-1, 1)
    n, cols = src.shape
    dst = np.empty((n, cols), order="F")
    load().orc_rotate(n, _ptr(basis), cols, _ptr(src), _ptr(dst))
    return dst


def trait_weights(values, h2, sigma2, trait=-1):
    values = _f(values)
    n = values.shape[0]
    d, k = np.empty(n), np.empty(n)
    st = _Status()
    _check(load().orc_trait_weights(n, _ptr(values), h2, sigma2, trait, _ptr(d), _ptr(k),
                                    ctypes.byref(st)), st)
    return d, k


def trait_context(values, xl_rot, y_rot, h2, sigma2, trait=-1):
    values, xl_rot, y_rot = _f(values), _f(xl_rot), _f(y_rot)
    n = values.shape[0]
    pm1 = xl_rot.shape[1] if xl_rot.ndim == 2 else 0
    v = np.empty(n)
    w_l = np.empty((n, max(pm1, 1)), order="F")
    s_tl = np.empty((max(pm1, 1), max(pm1, 1)), order="F")
    b_t = np.empty(max(pm1, 1))
    st = _Status()
    _check(load().orc_trait_context(n, pm1, _ptr(values), _ptr(xl_rot), _ptr(y_rot), h2, sigma2,
                                    trait, _ptr(v), _ptr(w_l), _ptr(s_tl), _ptr(b_t),
                                    ctypes.byref(st)), st)
    return {"v": v, "w_l": w_l[:, :pm1], "s_tl": s_tl[:pm1, :pm1], "b_t": b_t[:pm1]}


def solve_partitioned(basis, values, xl, xr, y, h2, sigma2):
    basis, values, xr, y = _f(basis), _f(values), _f(xr), _f(y)
    n = values.shape[0]
    xl = _f(xl).reshape(n, -1)
    pm1 = xl.shape[1]
    out = np.empty(pm1 + 1)
    st = _Status()
    _check(load().orc_solve_partitioned(n, pm1, _ptr(basis), _ptr(values), _ptr(xl), _ptr(xr),
                                        _ptr(y), h2, sigma2, _ptr(out), ctypes.byref(st)), st)
    return out


def solve_single(basis, values, x, y, h2, sigma2):
    basis, values, x, y = _f(basis), _f(values), _f(x), _f(y)
    n, p = x.shape
    out = np.empty(p)
    st = _Status()
    _check(load().orc_solve_single(n, p, _ptr(basis), _ptr(values), _ptr(x), _ptr(y), h2, sigma2,
                                   _ptr(out), ctypes.byref(st)), st)
    return out


def cholesky_solve(phi, x, y, h2, sigma2):
    phi, x, y = _f(phi), _f(x), _f(y)
    if x.ndim == 1:
        x = x.reshape(-1, 1)
    n, p = x.shape
    out = np.empty(p)
    st = _Status()
    _check(load().orc_cholesky_solve(n, p, _ptr(phi), _ptr(x), _ptr(y), h2, sigma2, _ptr(out),
                                     ctypes.byref(st)), st)
    return out


def cholesky_cells(phi, xl, snps, traits, h2, sigma2, cells_i, cells_j):
    """Cholesky-oracle b for the sampled cells; returns (k, p)."""
    phi, snps, traits = _f(phi), _f(snps), _f(traits)
    n = phi.shape[0]
    xl = _f(xl).reshape(n, -1)
    p = xl.shape[1] + 1
    m, t = snps.shape[1], traits.shape[1]
    ci = np.ascontiguousarray(cells_i, dtype=np.int64)
    cj = np.ascontiguousarray(cells_j, dtype=np.int64)
    out = np.empty((ci.shape[0], p))
    h2, sigma2 = _f(h2), _f(sigma2)
    st = _Status()
    _check(load().orc_cholesky_cells(n, p, m, t, _ptr(phi), _ptr(xl), _ptr(snps), _ptr(traits),
                                     _ptr(h2), _ptr(sigma2), ci.shape[0], _ptr(ci), _ptr(cj),
                                     _ptr(out), ctypes.byref(st)), st)
    return out


def compute_grid(values, xl_rot, snps_rot, traits_rot, h2, sigma2, workers=1, mbb=0, tbb=0,
                 layout="numpy"):
    """compute_tile over the whole grid from rotated operands; b as (m, t, p)."""
    values, snps_rot, traits_rot = _f(values), _f(snps_rot), _f(traits_rot)
    n = values.shape[0]
    xl_rot = _f(xl_rot).reshape(n, -1)
    p = xl_rot.shape[1] + 1
    m, t = snps_rot.shape[1], traits_rot.shape[1]
    h2, sigma2 = _f(h2), _f(sigma2)
    shape = (m, t, p) if layout == "numpy" else (t, m, p)
    out = np.empty(shape)
    st = _Status()
    _check(load().orc_compute_grid(n, p, m, t, _ptr(values), _ptr(xl_rot), _ptr(snps_rot),
                                   _ptr(traits_rot), _ptr(h2), _ptr(sigma2), mbb, tbb, workers,
                                   0 if layout == "numpy" else 1, _ptr(out), ctypes.byref(st)), st)
    return out


def solve_grid(kinship, xl, snps, traits, h2, sigma2, workers=1):
    """In-core restatement of gwgrid.solve_grid: b as (m, t, p)."""
    kinship, snps, traits = _f(kinship), _f(snps), _f(traits)
    n = kinship.shape[0]
    xl = _f(xl).reshape(n, -1)
    p = xl.shape[1] + 1
    m, t = snps.shape[1], traits.shape[1]
    h2, sigma2 = _f(h2), _f(sigma2)
    out = np.empty((m, t, p))
    st = _Status()
    _check(load().orc_solve_grid(n, p, m, t, _ptr(kinship), _ptr(xl), _ptr(snps), _ptr(traits),
                                 _ptr(h2), _ptr(sigma2), workers, 0, _ptr(out), ctypes.byref(st)),
           st)
    return out


def cell_flops(n: int, p: int) -> int:
    return int(load().orc_cell_flops(n, p))
