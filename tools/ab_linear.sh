#!/bin/bash
# A/B timing of engine builds on the c1 bench step (no CPU leg, no e2e):
#   LIBS="tools/_exp/libA.so tools/_exp/libB.so" REPS=2 [ARGS="--option i8_cluster=4"] bash tools/ab_linear.sh
for rep in $(seq ${REPS:-2}); do
for lib in ${LIBS}; do
  timeout 300 python - "$lib" ${ARGS:-} <<'PY' > gpurun_out/ab_$(basename $lib).log 2>&1
import sys, runpy
from paper_1210_7683_b200 import _native as nat
nat.LIB_PATH = sys.argv[1]
sys.argv = ["bench.py", "--steps", "20", "--warmup", "3", "--no-cpu", "--no-alt-coding", "--no-e2e"] + sys.argv[2:]
runpy.run_path("bench.py", run_name="__main__")
PY
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$(basename $lib).log').read().strip().splitlines()[-1]); b=d['roofline']['step_breakdown_ms']; print('$(basename $lib)', round(d['ms_per_step'],4), ' '.join('%s=%.4f' % (k.split()[0], v) for k, v in b.items()))" || tail -5 gpurun_out/ab_$(basename $lib).log
done
done
