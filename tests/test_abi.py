"""The C-ABI library loads and exports every symbol include/gwgrid_cuda.h
declares (no compute calls: this runs without a GPU)."""
import ctypes
import os
import re

import numpy as np
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


def test_struct_layouts_match_header(tmp_path):
    """sizeof / offsetof of every ABI struct, from the C compiler reading
    include/gwgrid_cuda.h, equal the ctypes mirrors."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc unavailable")
    fields = {"gwg_status": nat.Status, "gwg_counters": nat.Counters,
              "gwg_run_options": nat.RunOptions}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, cls in fields.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    for cname, cls in fields.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)


def test_cell_hash_matches_host_checksum():
    """gwg_cell_hash (the device checksum's term) equals the numpy
    recomputation used to check downloaded grids."""
    from paper_1210_7683_b200.checksum import grid_checksum

    rng = np.random.default_rng(5)
    b = rng.standard_normal((7, 5, 3))
    lib = nat.load()
    want = 0
    for i in range(7):
        for j in range(5):
            for c in range(3):
                bits = int(b[i, j, c:c + 1].view(np.uint64)[0])
                want = (want + lib.gwg_cell_hash(100 + i, j, c, bits)) & (2**64 - 1)
    assert grid_checksum(b, i0=100) == want
    assert grid_checksum(b.transpose(1, 0, 2).copy(), i0=100, layout="stream") == want
    # order independence: any split of the SNP axis sums to the same value
    parts = (grid_checksum(b[:3], i0=100) + grid_checksum(b[3:], i0=103)) & (2**64 - 1)
    assert parts == want
    b2 = b.copy()
    b2[3, 2, 1] = np.nextafter(b2[3, 2, 1], np.inf)  # one ulp anywhere changes it
    assert grid_checksum(b2, i0=100) != want


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
