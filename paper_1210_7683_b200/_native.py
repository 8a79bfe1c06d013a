"""ctypes binding of libgwgrid_cuda.so (the C ABI in include/gwgrid_cuda.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1210_7683_b200/csrc``).  There is no fallback: if the library is
missing, importing the engine raises immediately.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GWG_LIB") or os.path.join(_HERE, "libgwgrid_cuda.so")

GWG_OK = 0
GWG_DIMENSION = 1
GWG_NON_SYMMETRIC = 2
GWG_BACKEND = 3
GWG_NOT_POSITIVE_DEFINITE = 4
GWG_IO = 5
GWG_INFEASIBLE_BUDGET = 6
GWG_CUDA = 7

GWG_HOST = 0
GWG_DEVICE = 1
GWG_LAYOUT_NUMPY = 0
GWG_LAYOUT_STREAM = 1
GWG_SNP_REAL = 0
GWG_SNP_GENOTYPES = 1
GWG_SNP_AUTO = 2
GWG_FORMAT_F64 = 0
GWG_FORMAT_I8 = 1

# gwg_option
OPTIONS = {"split": 1, "sbr_direct": 2, "real_split": 3, "i8_cluster": 4, "sbr_cfg": 5}

# Every symbol include/gwgrid_cuda.h declares (checked by tests/test_abi.py).
EXPORTED_SYMBOLS = (
    "gwg_version",
    "gwg_engine_create",
    "gwg_engine_destroy",
    "gwg_eigendecompose",
    "gwg_set_kinship",
    "gwg_set_spectrum",
    "gwg_set_covariates",
    "gwg_set_traits",
    "gwg_solve_snp_slab",
    "gwg_run_grid",
    "gwg_set_snp_coding",
    "gwg_get_counters",
    "gwg_reset_counters",
    "gwg_synchronize",
    "gwg_compute_stream",
    "gwg_default_slab_snps",
    "gwg_verify_grid",
    "gwg_stream_info",
    "gwg_set_traits_file",
    "gwg_run_grid_files",
    "gwg_exp_sum_design",
    "gwg_gen_genotypes",
    "gwg_gen_normals",
    "gwg_gen_uniform",
    "gwg_set_option",
    "gwg_get_option",
    "gwg_cell_hash",
    "gwg_wait_stream",
    "gwg_signal_stream",
    "gwg_group_create",
    "gwg_group_destroy",
    "gwg_group_size",
    "gwg_group_engine",
    "gwg_group_set_spectrum",
    "gwg_group_set_covariates",
    "gwg_group_set_traits",
    "gwg_group_set_snp_coding",
    "gwg_group_set_option",
    "gwg_group_shards",
    "gwg_group_run_grid",
)


class Status(ctypes.Structure):
    _fields_ = [
        ("code", ctypes.c_int32),
        ("snp_index", ctypes.c_int64),
        ("trait_index", ctypes.c_int64),
        ("msg", ctypes.c_char * 256),
    ]


class Counters(ctypes.Structure):
    _fields_ = [
        ("preloop_flops", ctypes.c_uint64),
        ("loop_flops", ctypes.c_uint64),
        ("grid_flops", ctypes.c_uint64),
        ("bytes_loaded", ctypes.c_uint64),
        ("bytes_stored", ctypes.c_uint64),
        ("context_builds", ctypes.c_uint64),
        ("kernel_launches", ctypes.c_uint64),
        ("grid_kernel_ms", ctypes.c_double),
        ("rotate_ms", ctypes.c_double),
        ("wall_ms", ctypes.c_double),
        ("linear_ms", ctypes.c_double),
        ("quad_ms", ctypes.c_double),
        ("sbr_flops", ctypes.c_uint64),
        ("sbr_terms", ctypes.c_int64),
        ("io_stall_ms", ctypes.c_double),
        ("checksum", ctypes.c_uint64),
        ("checksum_cells", ctypes.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


# int32_t (*gwg_result_sink)(void* user, int64_t i0, int64_t rows, const double* cells)
RESULT_SINK = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                               ctypes.c_void_p)


class RunOptions(ctypes.Structure):
    _fields_ = [
        ("mb", ctypes.c_int64),
        ("layout", ctypes.c_int32),
        ("double_buffer", ctypes.c_int32),
        ("snp_format", ctypes.c_int32),
        ("checksum", ctypes.c_int32),
        ("i0", ctypes.c_int64),
        ("ldb", ctypes.c_int64),
        ("sink", RESULT_SINK),
        ("sink_user", ctypes.c_void_p),
        ("ring", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


_lib = None


def load() -> ctypes.CDLL:
    """Load the native library once; raise loudly when it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    I32, I64, U64, D = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    S = ctypes.POINTER(Status)
    sig = {
        "gwg_version": (ctypes.c_char_p, []),
        "gwg_engine_create": (P, [I32, I64, I64, S]),
        "gwg_engine_destroy": (None, [P]),
        "gwg_set_spectrum": (I32, [P, P, P, I32, S]),
        "gwg_eigendecompose": (I32, [I32, I64, P, I32, P, P, I32, S]),
        "gwg_set_kinship": (I32, [P, P, I32, S]),
        "gwg_set_covariates": (I32, [P, P, I32, S]),
        "gwg_set_traits": (I32, [P, I64, P, P, P, I32, I32, S]),
        "gwg_solve_snp_slab": (I32, [P, I64, I64, P, I32, I32, P, I32, I32, I64, S]),
        "gwg_run_grid": (I32, [P, I64, P, P, ctypes.POINTER(RunOptions),
                               ctypes.POINTER(Counters), S]),
        "gwg_verify_grid": (I32, [I32, I64, I64, I64, I64, P, P, P, P, P, P, P, P,
                                  ctypes.POINTER(D), S]),
        "gwg_stream_info": (I32, [ctypes.c_char_p, ctypes.POINTER(I32), ctypes.POINTER(I64),
                                  ctypes.POINTER(I32), S]),
        "gwg_set_traits_file": (I32, [P, ctypes.c_char_p, S]),
        "gwg_run_grid_files": (I32, [P, ctypes.c_char_p, I32, ctypes.c_char_p,
                                     ctypes.POINTER(RunOptions), ctypes.POINTER(Counters), S]),
        "gwg_set_snp_coding": (I32, [P, I32, S]),
        "gwg_get_counters": (I32, [P, ctypes.POINTER(Counters)]),
        "gwg_reset_counters": (None, [P]),
        "gwg_synchronize": (I32, [P, S]),
        "gwg_compute_stream": (P, [P]),
        "gwg_default_slab_snps": (I64, [P, I64]),
        "gwg_gen_genotypes": (None, [U64, I32, I64, I64, I64, I32, P, I64]),
        "gwg_gen_normals": (None, [U64, I32, I64, I64, I64, P, I64]),
        "gwg_gen_uniform": (None, [U64, I32, I64, D, D, P]),
        "gwg_exp_sum_design": (I32, [D, D, I32, I32, P, P, P]),
        "gwg_set_option": (I32, [P, I32, I64, S]),
        "gwg_get_option": (I32, [P, I32, ctypes.POINTER(I64), S]),
        "gwg_cell_hash": (U64, [I64, I64, I64, U64]),
        "gwg_wait_stream": (I32, [P, P, S]),
        "gwg_signal_stream": (I32, [P, P, S]),
        "gwg_group_create": (P, [ctypes.POINTER(I32), I32, I64, I64, S]),
        "gwg_group_destroy": (None, [P]),
        "gwg_group_size": (I32, [P]),
        "gwg_group_engine": (P, [P, I32]),
        "gwg_group_set_spectrum": (I32, [P, P, P, I32, S]),
        "gwg_group_set_covariates": (I32, [P, P, I32, S]),
        "gwg_group_set_traits": (I32, [P, I64, P, P, P, I32, I32, S]),
        "gwg_group_set_snp_coding": (I32, [P, I32, S]),
        "gwg_group_set_option": (I32, [P, I32, I64, S]),
        "gwg_group_shards": (I32, [P, I64, ctypes.POINTER(I64)]),
        "gwg_group_run_grid": (I32, [P, I64, P, P, ctypes.POINTER(RunOptions),
                                     ctypes.POINTER(Counters), S]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
