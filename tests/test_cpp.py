"""Runs the C++ host-mirror test program (tests/cpp/test_engine.cpp) on the GPU."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "_build", "test_engine")


@pytest.mark.gpu
def test_cpp_host_mirror():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", os.path.join(HERE, "cpp")], check=True)
    res = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failed" in res.stdout


def test_cpp_host_mirror_builds():
    """The C++ mirror compiles and links against the C ABI (no GPU needed)."""
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
    assert os.path.exists(BIN)
