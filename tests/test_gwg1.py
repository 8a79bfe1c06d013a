"""GWG1 stream format (proj/include/gwgrid/stream.hpp:15-41): host-side codec
checks (CPU) and the engine's file legs against the in-memory engine (GPU)."""
import ctypes
import os

import numpy as np
import pytest

import paper_1210_7683_b200 as gw
from paper_1210_7683_b200 import _native as nat
from paper_1210_7683_b200 import datagen, gwg1


def test_header_byte_layout_matches_reference_spec():
    h = gwg1.encode_header(gwg1.KIND_RESULT, (7, 5, 4), complete=False)
    assert len(h) == 64 and h[:4] == b"GWG1"
    assert h[4:6] == b"\x01\x00"          # version 1, little endian
    assert h[6] == 3 and h[7] == 0        # kind result, float64
    assert int.from_bytes(h[8:16], "little") == 7
    assert int.from_bytes(h[16:24], "little") == 5
    assert int.from_bytes(h[24:32], "little") == 4
    assert h[32] == 0 and h[33] == 1      # layout 0, incomplete
    assert h[34:] == bytes(30)


def test_round_trip_and_rejections(tmp_path):
    rng = np.random.default_rng(0)
    snps = rng.standard_normal((9, 6))
    p = str(tmp_path / "snps.gwg")
    gwg1.write_snp_stream(p, snps)
    assert np.array_equal(gwg1.read_columns(p), snps)
    with pytest.raises(gw.IoError, match="expected a trait stream"):
        gwg1.read_header(p, gwg1.KIND_TRAIT)
    raw = bytearray(open(p, "rb").read())
    for patch, msg in (((0, b"XWG1"), "bad magic"), ((4, b"\x02"), "version"),
                       ((33, b"\x01"), "never finalized"), ((7, b"\x01"), "element type")):
        bad = bytearray(raw)
        bad[patch[0]:patch[0] + len(patch[1])] = patch[1]
        q = str(tmp_path / "bad.gwg")
        open(q, "wb").write(bytes(bad))
        with pytest.raises(gw.IoError, match=msg):
            gwg1.read_header(q)
    q = str(tmp_path / "short.gwg")
    open(q, "wb").write(bytes(raw[:-8]))
    with pytest.raises(gw.IoError, match="header promises"):
        gwg1.read_header(q)


def test_native_stream_info_reads_headers_without_gpu(tmp_path):
    p = str(tmp_path / "t.gwg")
    gwg1.write_trait_stream(p, np.ones((5, 3)), [0.1, 0.2, 0.3], [1, 1, 1])
    kind, dims, complete = ctypes.c_int32(), (ctypes.c_int64 * 3)(), ctypes.c_int32()
    st = nat.Status()
    rc = nat.load().gwg_stream_info(p.encode(), ctypes.byref(kind), dims, ctypes.byref(complete),
                                    ctypes.byref(st))
    assert rc == 0 and kind.value == 2 and list(dims) == [5, 3, 0] and complete.value == 1


@pytest.mark.gpu
@pytest.mark.parametrize("coding", ["real", "genotypes"])
def test_file_legs_match_in_memory_engine(tmp_path, coding):
    ds = datagen.generate(300, 4, 1111, 45, seed=5)
    basis, values = gw.eigendecompose(ds["kinship"])
    snp_path, trait_path = str(tmp_path / "snps.gwg"), str(tmp_path / "traits.gwg")
    out_path = str(tmp_path / "b.gwg")
    gwg1.write_snp_stream(snp_path, ds["snps"])
    gwg1.write_trait_stream(trait_path, ds["traits"], ds["h2"], ds["sigma2"])
    with gw.Engine(300, 4) as eng:
        eng.set_spectrum(basis, values)
        eng.set_covariates(ds["xl"])
        eng.set_snp_coding(coding)
        eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
        mem = eng.run_grid(ds["snps"])
        eng.set_traits_file(trait_path)
        for mb in (0, 100, 1111):
            c = eng.run_grid_files(snp_path, out_path, mb=mb)
            got = gwg1.read_result(out_path)
            assert np.array_equal(got, mem)
        assert c["bytes_stored"] >= 1111 * 45 * 4 * 8
        # the file leg against the oracle (restated compute_tile), not only
        # against the in-memory engine
        from oracle import oracle as orc
        from tests.test_gpu_parity import assert_parity

        ref = orc.compute_grid(values, orc.rotate(basis, ds["xl"]), orc.rotate(basis, ds["snps"]),
                               orc.rotate(basis, ds["traits"]), ds["h2"], ds["sigma2"], workers=8)
        assert_parity(gwg1.read_result(out_path), ref)
        # a rotated SNP stream (the reference's preloop output) gives the same cells
        rot_path = str(tmp_path / "rot.gwg")
        gwg1.write_snp_stream(rot_path, basis.T @ ds["snps"])
        eng.run_grid_files(rot_path, out_path, rotated=True)
        rel = np.abs(gwg1.read_result(out_path) - mem).max() / np.abs(mem).max()
        assert rel < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("coding", ["real", "genotypes"])
def test_failed_run_leaves_unreadable_output(tmp_path, coding):
    """test_grid.cpp:766-771: no output survives as a readable stream."""
    ds = datagen.generate(40, 3, 10, 4, seed=6)
    snps = ds["snps"].copy()
    snps[:, 3] = 0.0
    snp_path, out_path = str(tmp_path / "snps.gwg"), str(tmp_path / "b.gwg")
    gwg1.write_snp_stream(snp_path, snps)
    with gw.Engine(40, 3) as eng:
        eng.set_spectrum(*gw.eigendecompose(ds["kinship"]))
        eng.set_covariates(ds["xl"])
        eng.set_snp_coding(coding)
        eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
        with pytest.raises(gw.NotPositiveDefiniteError) as e:
            eng.run_grid_files(snp_path, out_path)
        assert (e.value.snp_index, e.value.trait_index) == (3, 0)
        with pytest.raises(gw.IoError, match="never finalized"):
            gwg1.read_result(out_path)
        with pytest.raises(gw.IoError, match="expected a variant stream"):
            gwg1.write_trait_stream(snp_path, ds["traits"], ds["h2"], ds["sigma2"])
            eng.run_grid_files(snp_path, out_path)
