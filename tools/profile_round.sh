#!/bin/bash
# Round profiling recipe (run under gpurun): the bench line, its launch list,
# and one full ncu capture of the hot kernels at config c1 (genotype coding:
# rotate_i8_kernel (rotation), gls_sbr_kernel x6 (4 for the factorised W build at
# p = 4, 2 for the factorised S_BR), linear_solve_kernel;
# real coding: gls_grid_kernel and rotate_kernel).
set -u
R=${1:-r01}
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 > gpurun_out/${R}_bench.log 2>&1
echo "bench rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu --no-alt-coding > gpurun_out/${R}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-alt-coding \
    > gpurun_out/${R}_ncu_launches.log 2>&1
echo "launches rc=$?"
python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-alt-coding > gpurun_out/${R}_plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gls_sbr|rotate_i8|linear_solve" -s 8 -c 8 \
    -o gpurun_out/${R}_kernels python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-alt-coding \
    > gpurun_out/${R}_ncu_full.log 2>&1
echo "full rc=$?"
