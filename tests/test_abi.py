"""The C-ABI library loads and exports every symbol include/gwgrid_cuda.h
declares (no compute calls: this runs without a GPU)."""
import ctypes
import os
import re

import pytest

from paper_1210_7683_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gwgrid_cuda.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gwg_[a-z_0-9]+)\s*\(", src)))


def test_header_matches_python_binding_list():
    assert declared_symbols() == sorted(nat.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = nat.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_version_string():
    assert nat.load().gwg_version().decode().startswith("gwgrid_cuda ")
    assert b"sm_100a" in nat.load().gwg_version()


def test_struct_layouts_match_header():
    # gwg_status: int32 code, int64 snp, int64 trait, char[256]
    assert ctypes.sizeof(nat.Status) == 8 + 8 + 8 + 256
    assert nat.Status.snp_index.offset == 8
    assert ctypes.sizeof(nat.Counters) == 7 * 8 + 5 * 8 + 2 * 8
    assert ctypes.sizeof(nat.RunOptions) == 16


def test_library_is_sm100a_code():
    """The shipped .so carries sm_100a SASS (cuobjdump is in the image)."""
    import shutil
    import subprocess

    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump unavailable")
    out = subprocess.run(["cuobjdump", "--list-elf", nat.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_engine_create_without_gpu_fails_cleanly():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    st = nat.Status()
    h = nat.load().gwg_engine_create(0, 16, 3, ctypes.byref(st))
    assert not h
    assert st.code == nat.GWG_CUDA
    assert st.msg


def test_bad_dimensions_rejected_before_device():
    st = nat.Status()
    assert not nat.load().gwg_engine_create(0, 4, 5, ctypes.byref(st))  # p > n
    assert st.code == nat.GWG_DIMENSION
    assert not nat.load().gwg_engine_create(0, 100, 33, ctypes.byref(st))  # p out of range
    assert st.code == nat.GWG_DIMENSION and b"1..32" in st.msg
