"""The device path against outputs of the REFERENCE ITSELF (-m gpu).

* tests/golden/ref_grids.npz: grids the reference's own sources produced in
  the build container (tests/golden/make_ref_golden.py; /root/reference does
  not exist on the GPU box).  Inputs regenerate bit-identically from the
  counter-based generator, so only seeds and outputs are stored.
* when the prebuilt reference library travelled with the repo
  (oracle/_ref/libgwgrid_ref.so: gwgrid's gls.cpp / grid.cpp / stream.cpp ...
  compiled against our Eigen stand-in), the reference's streamed CT engine is
  also run live on the box's host cores at n = 1000, p = 4 and compared with
  the device on every cell, and its GWG1 reader decodes the result stream our
  engine's file leg wrote.

Tolerances as in tests/test_gpu_parity.py: norm-wise <= 1e-10 per cell,
components within 1e-8 floored at 1e-6 of the cell norm (typical 1e-14).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1210_7683_b200 as gw  # noqa: E402
from oracle import ref  # noqa: E402
from oracle.parity import parity_metrics  # noqa: E402
from paper_1210_7683_b200 import datagen, gwg1  # noqa: E402
from tests.golden import make_ref_golden as golden  # noqa: E402
from tests.test_gpu_parity import assert_parity  # noqa: E402

have_ref_build = pytest.mark.skipif(not os.path.exists(ref.LIB_PATH),
                                    reason="prebuilt reference library did not travel")


def codings(kind):
    # genotype codes run the default (auto -> exact int8 split grid), the
    # explicit genotype coding and the all-FP64 path; real values only the latter
    return ("auto", "genotypes", "real") if kind == "codes" else ("auto", "real")


@pytest.mark.parametrize("name", sorted(golden.CASES))
def test_device_matches_reference_goldens(name):
    want = golden.load()[name]
    ds = golden.inputs(name)
    kind = golden.CASES[name][5]
    for coding in codings(kind):
        res = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                            ds["sigma2"], snp_coding=coding)
        assert res["b"].shape == want["b"].shape
        assert_parity(res["b"], want["b"])
        ci, cj = golden.cholesky_cells(name)
        rel = np.linalg.norm(res["b"][ci, cj] - want["chol"], axis=1) / np.linalg.norm(
            want["chol"], axis=1)
        assert rel.max() <= 1e-9, (coding, rel.max())


LIVE_SHAPES = {
    # configs[0]/[1]'s n and p
    "c0_c1": (1000, 4, 3000, 300, 77),
    # configs[3]: many traits per SNP slab (t >> m)
    "c3": (1000, 4, 256, 4096, 78),
    # configs[4]: n = 2000, p = 20 (one trait per int8 tile, precomputed L^-1 solve)
    "c4": (2000, 20, 600, 256, 79),
}


@have_ref_build
@pytest.mark.parametrize("coding", ["auto", "real"])
@pytest.mark.parametrize("shape", sorted(LIVE_SHAPES))
def test_device_matches_live_reference_every_cell(shape, coding):
    """The reference's streamed CT engine (its own sources, built in the
    container) run live on the box's host cores against the device, every
    cell, at the n / p / t regimes of BASELINE's configs."""
    n, p, m, t, seed = LIVE_SHAPES[shape]
    ds = datagen.generate(n, p, m, t, seed=seed)
    want = ref.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                          ds["sigma2"], workers=min(16, os.cpu_count() or 1))
    got = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"],
                        snp_coding=coding)["b"]
    pm = parity_metrics(got, want)
    print(f"device ({coding}) vs live reference build, {shape} {m * t} cells: "
          f"normwise {pm['normwise_max']:.3e} floored {pm['floored_componentwise_max']:.3e} "
          f"raw {pm['raw_componentwise_max']:.3e}")
    assert pm["normwise_max"] <= 1e-10, pm
    assert pm["floored5_componentwise_max"] <= 1e-8, pm
    assert pm["n_floored_over_1e-8"] <= 1, pm


@have_ref_build
@pytest.mark.parametrize("coding", ["genotypes", "real"])
def test_reference_reader_decodes_engine_result_stream(tmp_path, coding):
    """stream.cpp:414-445 / 83-200: the result stream written by
    gwg_run_grid_files is a valid, complete kind-3 stream for the reference's
    reader, cell for cell; the reference's engine over the same input files
    agrees with it."""
    ds = datagen.generate(120, 3, 257, 19, seed=13)
    snp_path, trait_path = str(tmp_path / "snps.gwg"), str(tmp_path / "traits.gwg")
    out_path, ref_out = str(tmp_path / "b.gwg"), str(tmp_path / "b_ref.gwg")
    gwg1.write_snp_stream(snp_path, ds["snps"])
    gwg1.write_trait_stream(trait_path, ds["traits"], ds["h2"], ds["sigma2"])
    with gw.Engine(120, 3) as eng:
        eng.set_spectrum(*gw.eigendecompose(ds["kinship"]))
        eng.set_covariates(ds["xl"])
        eng.set_snp_coding(coding)
        eng.set_traits_file(trait_path)
        eng.run_grid_files(snp_path, out_path, mb=100)
    decoded = ref.read_result(out_path)
    assert np.array_equal(decoded, gwg1.read_result(out_path))
    ref.run_grid_files(ds["kinship"], ds["xl"], snp_path, trait_path, ref_out, workers=2)
    assert_parity(decoded, ref.read_result(ref_out))


DROPIN = os.path.join(os.path.dirname(ref.LIB_PATH), "dropin_run_grid")


@pytest.mark.skipif(not os.path.exists(DROPIN), reason="prebuilt drop-in program did not travel")
@pytest.mark.parametrize("shape", [
    "96 4 300 50 128 20 7 real",        # ragged slabs, 3 trait passes
    "200 4 500 300 256 300 8 codes",    # raw genotype codes -> exact int8 path, t >= 256
    "120 1 64 9 64 4 9 real",           # p = 1
    "1000 4 2000 100 512 100 10 real",  # configs 0/1's n and p
    "150 12 90 40 90 16 11 codes",      # p = 12, trait passes
])
def test_dropin_inside_reference_run_grid(tmp_path, shape):
    """INTEGRATION.md section 1 as a program (oracle/refbuild/dropin_run_grid.cpp):
    the reference's own run_grid traversal (its generator, GWG1 streams,
    TileParams, ResultTile, result writer, compiled from its sources) with
    load_pass -> gwg_set_traits and compute_tile -> gwg_solve_snp_slab, against
    the reference's run_grid on the CPU: every cell norm-wise <= 1e-10, the same
    NotPositiveDefiniteError coordinates for a zero variant column, and no
    readable output after the failure."""
    import subprocess

    run = subprocess.run([DROPIN, str(tmp_path)] + shape.split(), capture_output=True, text=True,
                         timeout=600)
    print(run.stdout)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "status=ok" in run.stdout


@have_ref_build
def test_cli_solves_a_reference_generated_dataset(tmp_path):
    """A gwgrid-dataset-1 directory written by the reference's own
    generate_dataset (datagen.cpp:263-315) goes through our CLI's solve and
    verify; the result stream equals the reference engine's over the same
    files to rounding."""
    import subprocess
    import sys

    from paper_1210_7683_b200 import cli

    d = tmp_path / "ds"
    ref.generate_dataset(d, 150, 4, 400, 30, seed=21)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

    def run(*args):
        r = subprocess.run([sys.executable, "-m", "paper_1210_7683_b200", *args], cwd=root,
                           capture_output=True, text=True, timeout=600)
        return r.returncode, dict(ln.split("=", 1) for ln in r.stdout.splitlines() if "=" in ln), r

    rc, kv, r = run("solve", "--data", str(d))
    assert rc == 0 and kv["status"] == "ok", r.stderr
    rc, kv2, r = run("verify", "--data", str(d), "--sample", "300")
    assert rc == 0 and kv2["status"] == "ok" and float(kv2["max_rel_err"]) < 1e-10, r.stdout
    man = cli.load_manifest(str(d))
    kin = gwg1.read_columns(man["kinship"], gwg1.KIND_OPERAND)
    xl = gwg1.read_columns(man["xl"], gwg1.KIND_OPERAND)
    ref_out = str(tmp_path / "b_ref.gwg")
    ref.run_grid_files(kin, xl, man["snps"], man["traits"], ref_out, workers=4)
    assert_parity(ref.read_result(kv["out"]), ref.read_result(ref_out))


REF_TOOL = os.path.join(os.path.dirname(ref.LIB_PATH), "gwgrid")


@pytest.mark.skipif(not os.path.exists(REF_TOOL), reason="prebuilt reference CLI did not travel")
@pytest.mark.parametrize("coding", ["auto", "real"])
def test_reference_cli_verifies_device_results(tmp_path, coding):
    """The reference's OWN command-line tool (proj/tools/gwgrid_main.cpp built
    against the stand-ins) generates a dataset; our CLI solves it on the
    device; the reference's `verify --exhaustive` (its CholeskyOracle over
    every cell, gwgrid_main.cpp:300-404) accepts the device's result stream.
    The other way round, our `verify` accepts the result stream the
    reference's `solve` wrote."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    d = str(tmp_path / "ds")

    def kv(stdout):
        return dict(ln.split("=", 1) for ln in stdout.splitlines() if "=" in ln)

    def theirs(*args):
        r = subprocess.run([REF_TOOL, *args], capture_output=True, text=True, timeout=600)
        return r.returncode, kv(r.stdout), r

    def ours(*args):
        r = subprocess.run([sys.executable, "-m", "paper_1210_7683_b200", *args], cwd=root,
                           capture_output=True, text=True, timeout=600)
        return r.returncode, kv(r.stdout), r

    rc, out, r = theirs("generate", "--n", "96", "--p", "4", "--m", "220", "--t", "24", "--seed", "3",
                        "--out", d)
    assert rc == 0 and out["status"] == "ok", r.stdout + r.stderr
    dev_out, cpu_out = str(tmp_path / "b_dev.gwg"), str(tmp_path / "b_cpu.gwg")
    rc, out, r = ours("solve", "--data", d, "--out", dev_out, "--snp-coding", coding)
    assert rc == 0 and out["status"] == "ok", r.stdout + r.stderr
    rc, out, r = theirs("verify", "--data", d, "--results", dev_out, "--exhaustive")
    print("reference verify of the device results:", out)
    assert rc == 0 and out["status"] == "ok", r.stdout + r.stderr
    assert float(out["max_rel_err"]) < 1e-10

    their_verify_keys = set(out)
    rc, out, r = theirs("solve", "--data", d, "--out", cpu_out, "--workers", "2")
    assert rc == 0 and out["status"] == "ok", r.stdout + r.stderr
    # our reports carry every key of the reference tool's (a script parsing
    # the reference's key=value lines keeps working)
    rc, mine, r = ours("solve", "--data", d, "--out", dev_out, "--snp-coding", coding)
    assert rc == 0 and set(out) <= set(mine), sorted(set(out) - set(mine))
    assert int(mine["mb"]) >= 1 and int(mine["tb"]) == 24 and float(mine["stall_fraction"]) >= 0.0
    rc, mine, r = ours("verify", "--data", d, "--results", dev_out, "--exhaustive")
    assert rc == 0 and their_verify_keys <= set(mine), sorted(their_verify_keys - set(mine))
    rc, out, r = ours("verify", "--data", d, "--results", cpu_out, "--sample", "400")
    assert rc == 0 and out["status"] == "ok" and float(out["max_rel_err"]) < 1e-10, r.stdout
    assert_parity(gwg1.read_result(dev_out), gwg1.read_result(cpu_out))
    # a corrupted cell is caught by the reference's verifier with exit code 3
    raw = np.fromfile(dev_out, dtype=np.uint8)
    cell = np.frombuffer(raw[gwg1.HEADER + 8 * 40:gwg1.HEADER + 8 * 41].tobytes(), dtype="<f8")[0]
    raw[gwg1.HEADER + 8 * 40:gwg1.HEADER + 8 * 41] = np.frombuffer(
        np.array([cell * 1.001 + 1e-3], dtype="<f8").tobytes(), dtype=np.uint8)
    bad = str(tmp_path / "b_bad.gwg")
    raw.tofile(bad)
    rc, out, r = theirs("verify", "--data", d, "--results", bad, "--exhaustive")
    assert rc == 3, r.stdout


@have_ref_build
def test_config0_full_size_device_vs_live_reference_every_cell():
    """BASELINE configs[0] at full size (n=1000, p=4, m=10,000, t=100: the
    reference's own CPU-runnable case), all 1e6 cells: the reference's streamed
    CT engine run live on the host against the device's default path."""
    ds = datagen.generate(1000, 4, 10_000, 100, seed=20260816)
    want = ref.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                          ds["sigma2"], workers=min(16, os.cpu_count() or 1))
    got = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"])["b"]
    pm = parity_metrics(got, want)
    print(f"c0 full size, device vs live reference build: normwise {pm['normwise_max']:.3e} "
          f"floored {pm['floored_componentwise_max']:.3e} raw {pm['raw_componentwise_max']:.3e} "
          f"({pm['n_raw_over_1e-8']} raw components over 1e-8 of {pm['components']})")
    assert pm["normwise_max"] <= 1e-10, pm
    assert pm["floored5_componentwise_max"] <= 1e-8, pm
    assert pm["n_floored_over_1e-8"] <= 4, pm
