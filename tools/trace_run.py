"""Run one c1 linear_solve launch against a LIN_TRACE build (tools/_exp/libtr.so)."""
import sys
sys.path.insert(0, ".")
from paper_1210_7683_b200 import _native as nat
nat.LIB_PATH = "tools/_exp/libtr.so"
import runpy
sys.argv = ["bench.py", "--steps", "1", "--warmup", "0", "--no-cpu", "--no-alt-coding", "--no-e2e"]
runpy.run_path("bench.py", run_name="__main__")
