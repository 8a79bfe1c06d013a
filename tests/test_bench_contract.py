"""The bench.py contract on the CPU: the reference arm (the oracle restatement
of the reference CPU path, runnable without a GPU) prints one JSON line with
the driver's keys, on the device arm's metric, unit and workload."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1", "--m", "200", "--t", "16", "--n", "64"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "config", "cpu_baseline", "e2e", "impl"):
        assert key in line, key
    assert line["impl"] == "reference" and line["unit"] == "GLS/s"
    assert line["higher_is_better"] is True and line["value"] > 0
    assert line["config"]["workload"] == "c1"
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["config"]["cells_per_step"] == 200 * 16  # the same grid as --m x --t


def test_reference_arm_loads_no_engine_code():
    """The reference arm times the CPU path only: inputs come from the oracle
    library's copy of the generator and the engine library is never mapped."""
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', "
            "'--warmup', '1', '--m', '50', '--t', '8', '--n', '32']; "
            "runpy.run_path('bench.py', run_name='__main__'); "
            "print('MAPS', sorted({l.split()[-1] for l in open('/proc/self/maps') "
            "if l.rstrip().endswith('.so')}))")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    maps = [ln for ln in r.stdout.splitlines() if ln.startswith("MAPS")][0]
    assert "libgls_oracle.so" in maps
    assert "libgwgrid_cuda.so" not in maps
