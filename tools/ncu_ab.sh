#!/bin/bash
# ncu a few metrics of one linear_solve launch for each lib in $LIBS
for lib in $LIBS; do
  name=$(basename $lib .so)
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none -k regex:linear_solve -s 2 -c 1 --csv \
    python - "$lib" > gpurun_out/ncuab_$name.csv 2>gpurun_out/ncuab_$name.err <<'PY'
import sys, runpy
from paper_1210_7683_b200 import _native as nat
nat.LIB_PATH = sys.argv[1]
sys.argv = ["bench.py", "--steps", "2", "--warmup", "1", "--no-cpu", "--no-alt-coding", "--no-e2e"]
runpy.run_path("bench.py", run_name="__main__")
PY
  echo "== $name"; grep -E "dram__|gpu__time|lts__" gpurun_out/ncuab_$name.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
