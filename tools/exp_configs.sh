#!/bin/bash
# tools/bench_configs.py (genotype coding) against alternative builds:
#   LIBS="paper_1210_7683_b200/libgwgrid_cuda.so tools/_exp/libK.so" CFGS=c1,c2 bash tools/exp_configs.sh
for lib in ${LIBS}; do
  GWG_SNP_CODING=genotypes timeout 600 python - "$lib" "${CFGS:-c1}" <<'PY'
import sys, runpy
from paper_1210_7683_b200 import _native as nat
nat.LIB_PATH = sys.argv[1]
lib = sys.argv[1]
sys.argv = ["bench_configs.py", "--configs", sys.argv[2]]
import json, io, contextlib
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    runpy.run_path("tools/bench_configs.py", run_name="__main__")
for line in buf.getvalue().splitlines():
    d = json.loads(line)
    print(lib.split("/")[-1], d["config"], round(d["ms_per_step"], 3), "rot", round(d["rotate_ms"], 3),
          "sbr", round(d["sbr_ms"], 3), "lin", round(d["linear_solve_ms"], 3))
PY
done
