#!/bin/bash
# Timing ablations of linear_solve (LIN_EXPERIMENT builds in tools/_exp/libK.so):
# runs bench.py against each library and prints the step breakdown.
for k in ${EXPS:-0 1 2 3 4}; do
  if [ $k = 0 ]; then lib=paper_1210_7683_b200/libgwgrid_cuda.so; else lib=tools/_exp/lib$k.so; fi
  timeout 120 python - "$lib" <<'PY' > gpurun_out/exp_$k.log 2>&1
import sys, runpy
from paper_1210_7683_b200 import _native as nat
nat.LIB_PATH = sys.argv[1]
sys.argv = ["bench.py", "--steps", "10", "--warmup", "3", "--no-cpu", "--no-alt-coding", "--no-e2e"]
runpy.run_path("bench.py", run_name="__main__")
PY
  echo "exp $k rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/exp_$k.log').read().strip().splitlines()[-1]); print($k, d['ms_per_step'], json.dumps(d['roofline']['step_breakdown_ms']))"
done
