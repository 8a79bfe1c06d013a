#!/bin/bash
# A/B timing of engine options on the c1 bench step (in-tree library):
#   OPTS="none i8_cluster=2 sbr_cfg=1" REPS=2 bash tools/ab_options.sh
for rep in $(seq ${REPS:-2}); do
for o in ${OPTS}; do
  extra=""; case $o in none) ;; layout=*) extra="--layout ${o#layout=}";; *) extra="--option $o";; esac
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-alt-coding --no-e2e $extra > gpurun_out/abo_$o.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abo_$o.log').read().strip().splitlines()[-1]); b=d['roofline']['step_breakdown_ms']; print('$o', round(d['ms_per_step'],4), ' '.join('%s=%.4f' % (k.split()[0], v) for k, v in b.items()))" || tail -3 gpurun_out/abo_$o.log
done
done
