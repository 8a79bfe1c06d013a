"""Pins the oracle (oracle/gls_oracle.cpp) to the REFERENCE ITSELF.  CPU only.

Two layers:
* the committed golden grids tests/golden/ref_grids.npz — outputs of the
  reference's own sources run in the build container
  (tests/golden/make_ref_golden.py) — against the oracle on regenerated
  inputs: always runs;
* the live reference build oracle/_ref/libgwgrid_ref.so (gwgrid's gls.cpp,
  grid.cpp, stream.cpp, pool.cpp, pipeline.cpp, types.cpp compiled where they
  lie under /root/reference against our Eigen stand-in, oracle/refbuild/):
  runs wherever that library exists or can be built, and skips elsewhere.

Tolerances: the oracle restates Eigen's reduction orders, the reference build
uses the stand-in's sequential loops, so agreement is to rounding: norm-wise
<= 1e-12 per cell (measured ~1e-14), components within 1e-9 of the cell norm
floor.  Error kinds and coordinates, the sign rule and everything the
reference promises bitwise (scheduler / tiling invariance) must match exactly.
"""
import os

import numpy as np
import pytest

from oracle import oracle as orc
from oracle import ref
from oracle.parity import parity_metrics
from paper_1210_7683_b200 import gwg1
from tests.golden import make_ref_golden as golden

live = pytest.mark.skipif(not ref.available(), reason="no reference sources / build here")


def normwise(got, want):
    return float((np.linalg.norm(got - want, axis=-1) / np.linalg.norm(want, axis=-1)).max())


def gen(n, p, m, t, seed):
    from paper_1210_7683_b200 import datagen

    return datagen.generate(n, p, m, t, seed=seed, lib=orc.load())


# ---- committed golden vectors (always) ----------------------------------

@pytest.mark.parametrize("name", sorted(golden.CASES))
def test_oracle_matches_reference_goldens(name):
    want = golden.load()[name]
    ds = golden.inputs(name, lib=orc.load())
    got = orc.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"],
                         workers=2)
    assert got.shape == want["b"].shape
    pm = parity_metrics(got, want["b"])
    assert pm["normwise_max"] <= 1e-12, pm
    assert pm["floored_componentwise_max"] <= 1e-9, pm
    # the reference's independent dense-Cholesky route at a few cells
    # (acceptance criterion 1, acceptance.cpp:110-163, bound 1e-8)
    ci, cj = golden.cholesky_cells(name)
    assert normwise(got[ci, cj], want["chol"]) <= 1e-10
    assert normwise(want["b"][ci, cj], want["chol"]) <= 1e-10


# ---- the live reference build --------------------------------------------

@live
@pytest.mark.parametrize("name", sorted(golden.CASES))
def test_committed_goldens_are_the_reference_output(name):
    """The committed file is what the reference build produces: bit for bit
    on the host that wrote it, to rounding on another CPU (OpenBLAS picks
    CPU-specific dgemm / dsyevd kernels for the rotation and the
    eigendecomposition under the reference's own code)."""
    want = golden.load()[name]
    got = golden.run_reference(name, lib=orc.load())
    assert got["b"].shape == want["b"].shape
    assert normwise(got["b"], want["b"]) <= 1e-12
    assert normwise(got["chol"], want["chol"]) <= 1e-12


@live
def test_eigendecomposition_matches_reference():
    """gls.cpp:16-46: ascending values, sign rule, symmetry gate."""
    rng = np.random.default_rng(5)
    a = rng.standard_normal((40, 40))
    phi = a @ a.T / 40 + np.eye(40)
    phi = 0.5 * (phi + phi.T)
    zr, lr = ref.eigendecompose(phi)
    zo, lo = orc.eigendecompose(phi)
    assert np.abs(lr - lo).max() <= 1e-13 * lo.max()
    assert np.abs(zr - zo).max() <= 1e-10  # same signs, same order
    bad = phi.copy()
    bad[3, 7] += 1e-6
    with pytest.raises(ref.RefError) as er:
        ref.eigendecompose(bad)
    with pytest.raises(orc.OracleError) as eo:
        orc.eigendecompose(bad)
    assert er.value.kind == "non_symmetric" and orc.CODES[eo.value.code] == "non_symmetric"


@live
@pytest.mark.parametrize("pm1", [0, 1, 3, 11])
def test_trait_context_matches_reference(pm1):
    """gls.cpp:48-103: d, k, v, W_L, S_TL (mirrored), b_T."""
    rng = np.random.default_rng(pm1)
    n = 57
    values = np.sort(rng.uniform(0.01, 4.0, n))
    xl = rng.standard_normal((n, pm1))
    y = rng.standard_normal(n)
    dr, kr = ref.trait_weights(values, 0.37, 1.9)
    do, ko = orc.trait_weights(values, 0.37, 1.9)
    assert np.array_equal(dr, do) and np.abs(kr - ko).max() <= 2e-16 * ko.max()
    cr = ref.trait_context(values, xl, y, 0.37, 1.9)
    co = orc.trait_context(values, xl, y, 0.37, 1.9)
    for key in ("v", "w_l", "s_tl", "b_t"):
        a, b = np.asarray(cr[key]), np.asarray(co[key]).reshape(np.shape(cr[key]))
        if a.size:
            assert np.abs(a - b).max() <= 1e-13 * max(1.0, np.abs(a).max()), key
    if pm1:
        assert np.array_equal(cr["s_tl"], cr["s_tl"].T)


@live
def test_weight_floor_error_matches_reference():
    """gls.cpp:58-76: a weight below the relative floor -> NPD at (-1, trait)."""
    values = np.array([-0.5, 0.2, 1.0, 3.0])
    with pytest.raises(ref.RefError) as er:
        ref.trait_weights(values, 0.9, 1.0, trait=6)
    with pytest.raises(orc.OracleError) as eo:
        orc.trait_weights(values, 0.9, 1.0, trait=6)
    assert er.value.kind == "not_positive_definite"
    assert (er.value.snp_index, er.value.trait_index) == (-1, 6)
    assert (eo.value.snp_index, eo.value.trait_index) == (-1, 6)
    assert str(er.value) == str(eo.value)


@live
@pytest.mark.parametrize("n,p,m,t,seed", [(24, 1, 9, 7, 1), (24, 24, 5, 3, 2), (50, 2, 1, 1, 3),
                                          (77, 5, 31, 13, 4), (130, 9, 17, 40, 5),
                                          (211, 13, 12, 9, 6), (96, 32, 6, 5, 7)])
def test_grids_match_reference(n, p, m, t, seed):
    """The oracle's solve_grid against the reference's streamed engine
    (bindings.cpp:115-190 -> grid.cpp:378-641) on ragged shapes, p = 1, n = p."""
    ds = gen(n, p, m, t, seed)
    want = ref.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                          ds["sigma2"], workers=2, mb=max(1, m // 2), tb=max(1, t // 3))
    got = orc.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"],
                         workers=2)
    pm = parity_metrics(got, want)
    # n = p interpolates: conditioning of the p x p system amplifies rounding
    bound = 1e-12 if n > p else 1e-7
    assert pm["normwise_max"] <= bound, pm


@live
def test_single_and_partitioned_solves_match_reference():
    """gls.cpp:134-186 and the Cholesky route gls.cpp:188-244."""
    ds = gen(83, 4, 6, 5, 11)
    basis, values = ref.eigendecompose(ds["kinship"])
    for i, j in [(0, 0), (5, 4), (2, 3)]:
        h2, s2 = float(ds["h2"][j]), float(ds["sigma2"][j])
        xr, y = ds["snps"][:, i], ds["traits"][:, j]
        pr = ref.solve_partitioned(basis, values, ds["xl"], xr, y, h2, s2)
        po = orc.solve_partitioned(basis, values, ds["xl"], xr, y, h2, s2)
        x = np.column_stack([ds["xl"], xr])
        sr = ref.solve_single(basis, values, x, y, h2, s2)
        so = orc.solve_single(basis, values, x, y, h2, s2)
        ch = ref.cholesky_cells(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                                ds["sigma2"], [i], [j])[0]
        for a in (po, sr, so, ch):
            assert np.linalg.norm(a - pr) <= 1e-12 * np.linalg.norm(pr)


@live
def test_cell_error_coordinates_match_reference():
    """gls.cpp:119-128 through grid.cpp:191-273: a zero variant column is not
    positive definite; the first failing cell in traversal order is reported."""
    ds = gen(40, 3, 12, 5, 9)
    ds["snps"][:, 7] = 0.0
    with pytest.raises(ref.RefError) as er:
        ref.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"])
    with pytest.raises(orc.OracleError) as eo:
        orc.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"])
    assert er.value.kind == "not_positive_definite"
    assert (er.value.snp_index, er.value.trait_index) == (7, 0)
    assert (eo.value.snp_index, eo.value.trait_index) == (7, 0)
    assert str(er.value) == str(eo.value)


@live
def test_reference_is_invariant_to_scheduler_and_tiling():
    """grid.hpp:27-31's promise, checked on the reference build itself (it
    also exercises the stand-in's block aliasing): ct / it / naive, workers,
    slab and block sizes, single vs double buffering — byte-identical."""
    ds = gen(48, 4, 37, 23, 21)
    args = (ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"])
    base, counters = ref.solve_grid(*args, return_counters=True)
    # the result grid plus the rotated variant stream the preloop transform writes
    assert counters["bytes_stored"] == 37 * 23 * 4 * 8 + 48 * 37 * 8
    assert counters["context_builds"] == 1
    for kw in (dict(scheduler="it", workers=3), dict(scheduler="naive"),
               dict(workers=4, mb=5, tb=4, mbb=2, tbb=3), dict(nb=1, mb=37, tb=1),
               dict(workers=2, mb=8, tb=6, double_buffer=False)):
        assert np.array_equal(ref.solve_grid(*args, **kw), base), kw


@live
def test_gwg1_codec_interoperates_with_reference_streams(tmp_path):
    """stream.cpp:83-445: files written by our codec are accepted by the
    reference's reader and engine, and the result stream it writes is decoded
    by our codec to the same bits as its own reader returns."""
    ds = gen(36, 3, 20, 11, 31)
    snps, traits, out = (str(tmp_path / f) for f in ("snps.gwg", "traits.gwg", "b.gwg"))
    gwg1.write_snp_stream(snps, ds["snps"])
    gwg1.write_trait_stream(traits, ds["traits"], ds["h2"], ds["sigma2"])
    counters = ref.run_grid_files(ds["kinship"], ds["xl"], snps, traits, out, workers=2, mb=7, tb=4)
    assert counters["context_builds"] == 3  # ceil(11 / 4) trait slabs
    got = gwg1.read_result(out)
    want = ref.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"])
    assert np.array_equal(got, want)
    # the rotated stream the reference wrote is a complete kind-1 stream for us
    rot = gwg1.read_columns(out + ".rot", gwg1.KIND_SNP)
    basis, _ = ref.eigendecompose(ds["kinship"])
    assert np.abs(rot - basis.T @ ds["snps"]).max() <= 1e-12
    # an unfinalized file of ours is rejected by the reference like by us
    with open(snps, "r+b") as f:
        f.seek(33)
        f.write(b"\x01")
    with pytest.raises(ref.RefError) as e:
        ref.run_grid_files(ds["kinship"], ds["xl"], snps, traits, out)
    assert e.value.kind == "io"


@live
def test_reference_acceptance_program_passes_here(tmp_path):
    """proj/tests/acceptance.cpp built from the reference's sources against
    the stand-in (oracle/_ref/gwgrid_acceptance) reproduces the reference's
    recorded run (proj/test_output.txt): criteria 1-5 and 8 pass with the same
    exact counts (loop flops, tiling 4x24, bytes_loaded=313728, min_tb=11).
    Criteria 6 (I/O stall fraction) and 7 (parallel speedup; it failed in the
    recorded run too, hardware_threads=1) are wall-clock measurements of the
    host: they pass here (stall 0.4%, speedup 3.7 on 8 cores) but are not
    asserted."""
    import subprocess

    exe = os.path.join(os.path.dirname(ref.LIB_PATH), "gwgrid_acceptance")
    if not os.path.exists(exe):
        ref.build()
    out = subprocess.run([exe], cwd=tmp_path, capture_output=True, text=True, timeout=600).stdout
    lines = {int(ln.split()[1]): ln for ln in out.splitlines() if ln.startswith("criterion ")}
    for k in (1, 2, 3, 4, 5, 8):  # 6 (stall fraction) and 7 (speedup) are wall-clock measurements
        assert ": PASS" in lines[k], lines[k]
    assert "loops_n64=124800 loops_n128=249600" in lines[2]
    assert "naive_transform_n64=1720320 naive_transform_n128=6881280" in lines[2]
    assert "mb=15 tb=1 tiles=4x24 bytes_loaded=313728 bitwise_identical=1" in lines[3]
    assert "configurations=8" in lines[4] and "all byte-identical" in lines[4]
    assert "min_tb=11 (expect 11)" in lines[5]
    err = float(lines[1].split("max_rel_err=")[1].split()[0])
    assert err < 1e-12  # recorded with real Eigen: 2.638e-14


# test cases / assertions of each reference unit-test file as they run here
# (every TEST_CASE of the file; SUBCASE leaves re-run their case like doctest)
REFERENCE_UNIT_TESTS = {"test_gls": 16, "test_grid": 18, "test_stream": 11, "test_pipeline": 10,
                        "test_datagen": 18, "test_tuner": 13, "test_cli": 10}


@live
@pytest.mark.parametrize("name", sorted(REFERENCE_UNIT_TESTS))
def test_reference_unit_tests_pass_here(name, tmp_path):
    """The reference's OWN unit tests (proj/tests/test_*.cpp, unmodified,
    compiled against the Eigen and doctest stand-ins) pass against this build
    of its sources: 96 test cases, ~3,100 assertions.  test_cli shells out to
    the reference's own command-line tool, built against the CLI11 stand-in
    (oracle/_ref/gwgrid)."""
    import subprocess

    exe = os.path.join(os.path.dirname(ref.LIB_PATH), "tests", name)
    if not os.path.exists(exe):
        ref.build()
    # test_pipeline / test_tuner hold a few wall-clock assertions (overlap vs
    # serial stall, measured rates): allow a loaded host two more attempts
    for attempt in range(3):
        run = subprocess.run([exe], cwd=tmp_path, capture_output=True, text=True, timeout=900)
        if run.returncode == 0 or name not in ("test_pipeline", "test_tuner", "test_cli"):
            break
    tail = run.stdout.strip().splitlines()[-2:]
    assert run.returncode == 0, run.stdout[-2000:]
    assert f"test cases: {REFERENCE_UNIT_TESTS[name]} | {REFERENCE_UNIT_TESTS[name]} passed | 0 failed" in tail[0]
    assert "0 failed" in tail[1]


@live
def test_compute_grid_in_core_matches_streamed_reference():
    """ref.compute_grid (the in-core composition bench.py times) against the
    reference's streamed route on the same operands."""
    ds = gen(90, 4, 70, 21, 17)
    basis, values = ref.eigendecompose(ds["kinship"])
    a = ref.compute_grid(basis, values, ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"],
                         workers=3, mb=16)
    b = ref.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"])
    assert normwise(a, b) <= 1e-13


@live
def test_dataset_directories_interoperate_with_reference(tmp_path):
    """gwgrid-dataset-1 (datagen.cpp:241-396) both ways: a directory written by
    the reference's generate_dataset is read by our manifest parser and codec;
    a directory written by our CLI's generate is accepted by the reference's
    load_manifest and read by its stream reader to the same payload sums."""
    from paper_1210_7683_b200 import cli

    theirs = tmp_path / "theirs"
    ref.generate_dataset(theirs, 40, 3, 25, 7, seed=5)
    man = cli.load_manifest(str(theirs))
    assert (man["n"], man["p"], man["m"], man["t"]) == (40, 3, 25, 7)
    kin = gwg1.read_columns(man["kinship"], gwg1.KIND_OPERAND)
    xl = gwg1.read_columns(man["xl"], gwg1.KIND_OPERAND)
    snps = gwg1.read_columns(man["snps"], gwg1.KIND_SNP)
    assert kin.shape == (40, 40) and xl.shape == (40, 2) and snps.shape == (40, 25)
    assert np.array_equal(kin, kin.T)
    dims, sums = ref.load_dataset(theirs / "manifest.txt")
    assert dims == (40, 3, 25, 7)
    assert np.isclose(sums[0], kin.sum(), rtol=1e-13) and np.isclose(sums[2], snps.sum(), rtol=1e-13)
    # the reference's engine over its own dataset == the oracle on what our codec read
    raw = np.fromfile(man["traits"], dtype="<f8", offset=gwg1.HEADER)
    traits, h2, s2 = raw[:40 * 7].reshape((40, 7), order="F"), raw[280:287], raw[287:294]
    out = str(tmp_path / "b.gwg")
    ref.run_grid_files(kin, xl, man["snps"], man["traits"], out)
    got = orc.solve_grid(kin, xl, snps, traits, h2, s2)
    assert normwise(got, ref.read_result(out)) <= 1e-12

    ours = str(tmp_path / "ours")
    ds = cli.write_dataset(ours, 36, 4, 20, 6, seed=9)
    dims, sums = ref.load_dataset(os.path.join(ours, "manifest.txt"))
    assert dims == (36, 4, 20, 6)
    want = [ds["kinship"].sum(), ds["xl"].sum(), ds["snps"].sum(), ds["traits"].sum(),
            ds["h2"].sum(), ds["sigma2"].sum()]
    assert np.allclose(sums, want, rtol=1e-12, atol=1e-12)


@live
def test_config0_every_cell_matches_reference():
    """BASELINE configs[0] (n=1000, p=4, m=10,000, t=100), all 1e6 cells:
    oracle vs the reference's streamed CT engine."""
    ds = gen(1000, 4, 10_000, 100, 20260816)
    workers = min(16, os.cpu_count() or 1)
    want = ref.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                          ds["sigma2"], workers=workers)
    got = orc.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"],
                         workers=workers)
    pm = parity_metrics(got, want)
    print("c0 oracle vs reference build:", pm)
    assert pm["normwise_max"] <= 1e-11, pm
    assert pm["floored_componentwise_max"] <= 1e-8, pm
