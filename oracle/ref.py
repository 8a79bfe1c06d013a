"""ctypes face of oracle/_ref/libgwgrid_ref.so — TEST INFRASTRUCTURE ONLY.

That library is the REFERENCE's own hot-path sources (gwgrid gls.cpp,
grid.cpp, stream.cpp, pool.cpp, pipeline.cpp, types.cpp) compiled where they
lie under /root/reference by oracle/refbuild/Makefile, against our stand-in for
<Eigen/Dense> (Eigen3 is absent from the image; see the stand-in's header for
what that carries over), behind the small C face oracle/refbuild/ref_capi.cpp.
The same Makefile builds the reference's acceptance program, its seven doctest
suites (doctest stand-in) and its command-line tool (CLI11 stand-in) into
oracle/_ref/ for tests/test_ref_pin.py and tests/test_gpu_ref_golden.py.
It is used to pin oracle/gls_oracle.cpp (tests/test_ref_pin.py) and to write
the golden vectors tests/golden/ref_*.npz (tests/golden/make_ref_golden.py).
Only tests/ may import this module.  /root/reference does not exist on the
GPU box: the GPU tests use the committed vectors, plus this PREBUILT library
when it travelled with the repo snapshot (it is git-ignored, not
gpurun-ignored); nothing there reads /root/reference.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import tempfile

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libgwgrid_ref.so")
REFERENCE_SRC = "/root/reference/proj/src"

SCHEDULERS = {"ct": 0, "it": 1, "naive": 2}
CODES = {1: "dimension", 2: "non_symmetric", 3: "backend", 4: "not_positive_definite",
         5: "io", 6: "error", 7: "other"}


class RefError(Exception):
    def __init__(self, code: int, msg: str, snp_index: int, trait_index: int):
        super().__init__(msg)
        self.code = code
        self.kind = CODES.get(code, "?")
        self.snp_index = snp_index
        self.trait_index = trait_index


class _Status(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("snp_index", ctypes.c_int64),
                ("trait_index", ctypes.c_int64), ("msg", ctypes.c_char * 256)]


_lib = None


def available() -> bool:
    """True when the reference build exists or can be made (sources present)."""
    return os.path.exists(LIB_PATH) or os.path.isdir(REFERENCE_SRC)


def build() -> str:
    subprocess.run(["make", "-s", "-C", os.path.join(_HERE, "refbuild")], check=True)
    return LIB_PATH


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        lib = ctypes.CDLL(LIB_PATH)
        P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        S, C = ctypes.POINTER(_Status), ctypes.c_char_p
        for name, args in {
            "ref_eigendecompose": [I64, P, P, P, S],
            "ref_trait_weights": [I64, P, D, D, I64, P, P, S],
            "ref_trait_context": [I64, I64, P, P, P, D, D, I64, P, P, P, P, S],
            "ref_solve_partitioned": [I64, I64, P, P, P, P, P, D, D, P, S],
            "ref_solve_single": [I64, I64, P, P, P, P, D, D, P, S],
            "ref_cholesky_cells": [I64, I64, I64, I64, P, P, P, P, P, P, I64, P, P, S],
            "ref_solve_grid": [I64, I64, I64, I64, P, P, P, P, P, P, I32, I32, I64, I64, I64, I64,
                               I64, I32, C, P, P, S],
            "ref_run_grid_files": [I64, I64, P, P, C, C, C, C, I32, I32, I64, I64, I64, I64, I64,
                                   I32, P, S],
            "ref_read_result": [C, P, P, I64, S],
            "ref_generate_dataset": [C, I64, I64, I64, I64, ctypes.c_uint64, D, S],
            "ref_load_dataset": [C, P, P, S],
            "ref_compute_grid": [I64, I64, I64, I64, P, P, P, P, P, P, P, I32, I64, I64, I64, P, S],
        }.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = I32
        _lib = lib
    return _lib


def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _check(rc: int, st: _Status) -> None:
    if rc != 0:
        raise RefError(st.code, st.msg.decode(errors="replace"), st.snp_index, st.trait_index)


def eigendecompose(phi):
    """gwgrid::eigendecompose_kinship (gls.cpp:16-46)."""
    phi = _f(phi)
    n = phi.shape[0]
    basis = np.empty((n, n), order="F")
    values = np.empty(n)
    st = _Status()
    _check(load().ref_eigendecompose(n, _ptr(phi), _ptr(basis), _ptr(values), ctypes.byref(st)), st)
    return basis, values


def trait_weights(values, h2, sigma2, trait=-1):
    """gwgrid::build_trait_weights (gls.cpp:48-79)."""
    values = _f(values)
    n = values.shape[0]
    d, k = np.empty(n), np.empty(n)
    st = _Status()
    _check(load().ref_trait_weights(n, _ptr(values), h2, sigma2, trait, _ptr(d), _ptr(k),
                                    ctypes.byref(st)), st)
    return d, k


def trait_context(values, xl_rot, y_rot, h2, sigma2, trait=-1):
    """gwgrid::build_trait_context (gls.cpp:81-103)."""
    values, y_rot = _f(values), _f(y_rot)
    n = values.shape[0]
    xl_rot = _f(xl_rot).reshape(n, -1, order="F")
    pm1 = xl_rot.shape[1]
    v, w_l = np.empty(n), np.empty((n, pm1), order="F")
    s_tl, b_t = np.empty((pm1, pm1), order="F"), np.empty(pm1)
    st = _Status()
    _check(load().ref_trait_context(n, pm1, _ptr(values), _ptr(xl_rot), _ptr(y_rot), h2, sigma2,
                                    trait, _ptr(v), _ptr(w_l), _ptr(s_tl), _ptr(b_t),
                                    ctypes.byref(st)), st)
    return {"v": v, "w_l": w_l, "s_tl": s_tl, "b_t": b_t}


def solve_partitioned(basis, values, xl, xr, y, h2, sigma2):
    """gwgrid::solve_partitioned_gls (gls.cpp:163-186)."""
    basis, values, xr, y = _f(basis), _f(values), _f(xr), _f(y)
    n = basis.shape[0]
    xl = _f(xl).reshape(n, -1, order="F")
    pm1 = xl.shape[1]
    out = np.empty(pm1 + 1)
    st = _Status()
    _check(load().ref_solve_partitioned(n, pm1, _ptr(basis), _ptr(values), _ptr(xl), _ptr(xr),
                                        _ptr(y), h2, sigma2, _ptr(out), ctypes.byref(st)), st)
    return out


def solve_single(basis, values, x, y, h2, sigma2):
    """gwgrid::solve_single_gls (gls.cpp:134-161)."""
    basis, values, y = _f(basis), _f(values), _f(y)
    n = basis.shape[0]
    x = _f(x).reshape(n, -1, order="F")
    p = x.shape[1]
    out = np.empty(p)
    st = _Status()
    _check(load().ref_solve_single(n, p, _ptr(basis), _ptr(values), _ptr(x), _ptr(y), h2, sigma2,
                                   _ptr(out), ctypes.byref(st)), st)
    return out


def cholesky_cells(phi, xl, snps, traits, h2, sigma2, cells_i, cells_j):
    """gwgrid::CholeskyOracle (gls.cpp:188-244) at the listed (i, j) cells."""
    phi, snps, traits = _f(phi), _f(snps), _f(traits)
    n = phi.shape[0]
    xl = _f(xl).reshape(n, -1, order="F")
    pm1 = xl.shape[1]
    h2, sigma2 = _f(h2), _f(sigma2)
    order = np.argsort(np.asarray(cells_j), kind="stable")
    cells = np.ascontiguousarray(
        np.stack([np.asarray(cells_i)[order], np.asarray(cells_j)[order]], axis=1), dtype=np.int64)
    got = np.empty((len(order), pm1 + 1))
    st = _Status()
    _check(load().ref_cholesky_cells(n, pm1, snps.shape[1], traits.shape[1], _ptr(phi), _ptr(xl),
                                     _ptr(snps), _ptr(traits), _ptr(h2), _ptr(sigma2), len(order),
                                     cells.ctypes.data, _ptr(got), ctypes.byref(st)), st)
    out = np.empty_like(got)
    out[order] = got
    return out


def solve_grid(kinship, xl, snps, traits, h2, sigma2, scheduler="ct", workers=1, nb=0, mb=0, tb=0,
               mbb=0, tbb=0, double_buffer=True, return_counters=False):
    """The reference's gwgrid.solve_grid route (python/bindings.cpp:115-190):
    operands staged to GWG1 files by its own writer, preloop_stream_transform +
    run_grid (or run_grid_naive), the result stream read back: b as (m, t, p)."""
    kinship, snps, traits = _f(kinship), _f(snps), _f(traits)
    n = kinship.shape[0]
    xl = _f(xl).reshape(n, -1, order="F")
    p = xl.shape[1] + 1
    m, t = snps.shape[1], traits.shape[1]
    h2, sigma2 = _f(h2), _f(sigma2)
    out = np.empty((m, t, p))
    counters = np.zeros(3, dtype=np.uint64)
    st = _Status()
    with tempfile.TemporaryDirectory(prefix="gwgrid_ref_") as work:
        _check(load().ref_solve_grid(n, p, m, t, _ptr(kinship), _ptr(xl), _ptr(snps), _ptr(traits),
                                     _ptr(h2), _ptr(sigma2), SCHEDULERS[scheduler], workers, nb, mb,
                                     tb, mbb, tbb, int(double_buffer), work.encode(), _ptr(out),
                                     counters.ctypes.data, ctypes.byref(st)), st)
    if return_counters:
        return out, {"bytes_loaded": int(counters[0]), "bytes_stored": int(counters[1]),
                     "context_builds": int(counters[2])}
    return out


def run_grid_files(kinship, xl, snps_path, traits_path, out_path, rotated_path=None,
                   scheduler="ct", workers=1, nb=0, mb=0, tb=0, mbb=0, tbb=0, double_buffer=True):
    """The reference's streamed engine over GWG1 files written by somebody
    else (our codec): precompute_grid, preloop_stream_transform, run_grid
    (grid.cpp:378-641)."""
    kinship = _f(kinship)
    n = kinship.shape[0]
    xl = _f(xl).reshape(n, -1, order="F")
    p = xl.shape[1] + 1
    rotated_path = rotated_path or str(out_path) + ".rot"
    counters = np.zeros(3, dtype=np.uint64)
    st = _Status()
    _check(load().ref_run_grid_files(n, p, _ptr(kinship), _ptr(xl), str(snps_path).encode(),
                                     str(traits_path).encode(), str(rotated_path).encode(),
                                     str(out_path).encode(), SCHEDULERS[scheduler], workers, nb, mb,
                                     tb, mbb, tbb, int(double_buffer), counters.ctypes.data,
                                     ctypes.byref(st)), st)
    return {"bytes_loaded": int(counters[0]), "bytes_stored": int(counters[1]),
            "context_builds": int(counters[2])}


def read_result(path):
    """A GWG1 result stream decoded by the reference's own reader
    (stream.cpp:83-445): b as (m, t, p)."""
    dims = np.zeros(3, dtype=np.int64)
    st = _Status()
    _check(load().ref_read_result(str(path).encode(), dims.ctypes.data, None, 0, ctypes.byref(st)),
           st)
    out = np.empty(tuple(int(d) for d in dims))
    _check(load().ref_read_result(str(path).encode(), dims.ctypes.data, _ptr(out), out.size,
                                  ctypes.byref(st)), st)
    return out


def compute_grid(basis, values, xl, snps, traits, h2, sigma2, workers=1, mb=8192, mbb=0, tbb=0):
    """run_grid's in-core traversal (grid.cpp:495-556) without the file legs,
    from UNROTATED operands and a given eigensystem: rotate X_L and the trait
    slab, build_trait_contexts, then per slab of mb variant columns
    transform_snp_slab + compute_tile (CT blocks, `workers` pool threads; the
    rotation's dgemm uses OpenBLAS's own threads).  b as (m, t, p)."""
    basis, values, snps, traits = _f(basis), _f(values), _f(snps), _f(traits)
    n = basis.shape[0]
    xl = _f(xl).reshape(n, -1, order="F")
    p = xl.shape[1] + 1
    m, t = snps.shape[1], traits.shape[1]
    h2, sigma2 = _f(h2), _f(sigma2)
    out = np.empty((m, t, p))
    st = _Status()
    _check(load().ref_compute_grid(n, p, m, t, _ptr(basis), _ptr(values), _ptr(xl), _ptr(snps),
                                   _ptr(traits), _ptr(h2), _ptr(sigma2), workers, min(mb, m), mbb,
                                   tbb, _ptr(out), ctypes.byref(st)), st)
    return out


def generate_dataset(directory, n, p, m, t, seed=1, condition=100.0):
    """gwgrid::generate_dataset (datagen.cpp:263-315): a gwgrid-dataset-1
    directory (manifest.txt + four GWG1 streams) from the reference's own
    generator."""
    st = _Status()
    _check(load().ref_generate_dataset(str(directory).encode(), n, p, m, t, seed, condition,
                                       ctypes.byref(st)), st)


def load_dataset(manifest_path):
    """gwgrid::load_manifest + read_dense on a dataset somebody else wrote:
    ((n, p, m, t), sums of the kinship / xl / snps / traits / h2 / sigma2
    payloads as the reference read them)."""
    dims = np.zeros(4, dtype=np.int64)
    sums = np.zeros(6)
    st = _Status()
    _check(load().ref_load_dataset(str(manifest_path).encode(), dims.ctypes.data, sums.ctypes.data,
                                   ctypes.byref(st)), st)
    return tuple(int(d) for d in dims), sums
