#!/bin/bash
# A/B timing of engine builds on tools/bench_configs.py configs:
#   LIBS="tools/_exp/libA.so tools/_exp/libB.so" CONFIGS=c2,c4 REPS=2 [ARGS="--option i8_cluster=4"] bash tools/ab_configs.sh
for rep in $(seq ${REPS:-2}); do
for lib in ${LIBS}; do
GWG_SNP_CODING=genotypes timeout 600 python - "$lib" ${ARGS:-} <<PY
import sys, runpy, io, contextlib, json
from paper_1210_7683_b200 import _native as nat
nat.LIB_PATH = sys.argv[1]
sys.argv = ["bench_configs.py", "--configs", "${CONFIGS:-c2,c4}", "--steps", "2"] + sys.argv[2:]
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    runpy.run_path("tools/bench_configs.py", run_name="__main__")
for line in buf.getvalue().splitlines():
    d = json.loads(line)
    print(nat.LIB_PATH.split("/")[-1], d["options"], d["config"], round(d["ms_per_step"], 3), "rot", round(d["rotate_ms"], 3), "sbr", round(d["sbr_ms"], 3), "lin", round(d["linear_solve_ms"], 3))
PY
done; done
