"""CLI contract (mirrors proj/tests/test_cli.cpp): exit codes 0/1/2/3 and the
final `status=` line (gwgrid_main.cpp:4-5, 34-37)."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args):
    r = subprocess.run([sys.executable, "-m", "paper_1210_7683_b200", *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    lines = r.stdout.strip().splitlines()
    kv = dict(line.split("=", 1) for line in lines if "=" in line)
    return r.returncode, kv, r


def test_generate_writes_a_dataset(tmp_path):
    rc, kv, _ = run("generate", "--n", "30", "--p", "3", "--m", "20", "--t", "4", "--out",
                    str(tmp_path / "d"))
    assert rc == 0 and kv["status"] == "ok"
    from paper_1210_7683_b200 import cli, gwg1

    man = cli.load_manifest(str(tmp_path / "d"))
    assert (man["n"], man["p"], man["m"], man["t"]) == (30, 3, 20, 4)
    assert gwg1.read_header(man["snps"], gwg1.KIND_SNP)["dims"][:2] == (30, 20)
    assert gwg1.read_header(man["kinship"], gwg1.KIND_OPERAND)["dims"][:2] == (30, 30)


def test_usage_errors_exit_2():
    rc, kv, _ = run("bogus")
    assert rc == 2 and kv["status"] == "usage"
    rc, kv, _ = run("generate", "--n", "2", "--p", "5", "--m", "1", "--t", "1", "--out", "/tmp/x")
    assert rc == 2 and kv["status"] == "usage"
    rc, kv, _ = run("tune")
    assert rc == 2 and kv["status"] == "usage"
    rc, kv, _ = run("verify", "--data", "/nonexistent", "--sample", "0")
    assert rc == 2 and kv["status"] == "usage"


def test_missing_dataset_is_a_runtime_error():
    rc, kv, r = run("solve", "--data", "/nonexistent")
    assert rc == 1 and kv["status"] == "error"
    assert "manifest" in r.stderr


@pytest.mark.gpu
def test_solve_verify_round_trip_and_failures(tmp_path):
    import paper_1210_7683_b200 as gw
    from paper_1210_7683_b200 import cli, gwg1

    d = str(tmp_path / "d")
    assert run("generate", "--n", "80", "--p", "4", "--m", "300", "--t", "12", "--out", d)[0] == 0
    rc, kv, r = run("solve", "--data", d)
    assert rc == 0 and kv["status"] == "ok", r.stderr
    b = gwg1.read_result(kv["out"])
    man = cli.load_manifest(d)
    ds = {k: gwg1.read_columns(man[k], kind) for k, kind in
          (("kinship", 4), ("xl", 4), ("snps", 1))}
    raw = np.fromfile(man["traits"], dtype="<f8", offset=64)
    traits = raw[:80 * 12].reshape((80, 12), order="F")
    ref = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], traits, raw[960:972], raw[972:])
    assert np.array_equal(b, ref["b"])
    rc, kv, _ = run("verify", "--data", d, "--sample", "200")
    assert rc == 0 and kv["status"] == "ok" and float(kv["max_rel_err"]) < 1e-10
    # the genotype-coded path on the same dataset agrees to rounding
    rc, kv, _ = run("solve", "--data", d, "--snp-coding", "genotypes", "--out",
                    os.path.join(d, "bg.gwg"))
    assert rc == 0 and kv["snp_coding"] == "genotypes"
    bg = gwg1.read_result(kv["out"])
    assert np.max(np.linalg.norm(bg - b, axis=2) / np.linalg.norm(b, axis=2)) < 1e-10
    rc, kv, _ = run("verify", "--data", d, "--exhaustive")
    assert rc == 0 and kv["mode"] == "exhaustive" and int(kv["checked"]) == 300 * 12
    # corrupt one cell (test_cli.cpp:199-226): verification fails with exit 3
    with open(os.path.join(d, "b.gwg"), "r+b") as f:
        f.seek(64 + (5 * 300 + 17) * 4 * 8 + 8)
        f.write(np.float64(123.0).tobytes())
    rc, kv, _ = run("verify", "--data", d, "--exhaustive")
    assert rc == 3 and kv["status"] == "verification-failed"
    assert (kv["worst_snp"], kv["worst_trait"]) == ("17", "5")
    # zero a SNP column (test_cli.cpp:228-247): solve fails with coordinates
    snps = ds["snps"].copy()
    snps[:, 9] = 0.0
    gwg1.write_snp_stream(man["snps"], snps)
    rc, kv, _ = run("solve", "--data", d)
    assert rc == 1 and kv["status"] == "error" and kv["error"] == "not-positive-definite"
    assert (kv["snp_index"], kv["trait_index"]) == ("9", "0")
    rc, kv, _ = run("bench", "--data", d)
    assert rc == 1  # the zero column makes every run fail as well
