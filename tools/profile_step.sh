#!/bin/bash
# Config-3 step profile of the final code (GPU box): launch list of the eager step, full captures
# of the trisolve + dense-tail kernels, and the default-command launch list.
#   bash tools/profile_step.sh <tag>
set -u
TAG=${1:-r2}
OUT=gpurun_out/prof
mkdir -p $OUT
NCU="ncu --clock-control none"
HN_PRESSURE_EAGER=1 $NCU --set full --import-source on -k "regex:sptrsv_super_kernel|tail_" --launch-skip 10 -c 5 -f \
  -o $OUT/${TAG}_c3_trisolve python tools/prof_step_eager.py 4 > $OUT/ncu_c3_trisolve.log 2>&1
python tools/ncu_summary.py report $OUT/${TAG}_c3_trisolve.ncu-rep $OUT/${TAG}_c3_trisolve_full > /dev/null 2>> $OUT/ncu_c3_trisolve.log
rm -f $OUT/${TAG}_c3_trisolve.ncu-rep
HN_PRESSURE_EAGER=1 $NCU --metrics gpu__time_duration.sum -c 4000 --csv --log-file $OUT/${TAG}_c3_step_launches.csv \
  python tools/prof_step_eager.py 6 > $OUT/ncu_c3_step.log 2>&1
python tools/ncu_summary.py launches $OUT/${TAG}_c3_step_launches.csv $OUT/${TAG}_c3_step_launches.md > /dev/null
$NCU --metrics gpu__time_duration.sum -c 6000 --csv --log-file $OUT/${TAG}_default_launches.csv \
  python bench.py --steps 2 --warmup 3 > $OUT/ncu_default.log 2>&1
python tools/ncu_summary.py launches $OUT/${TAG}_default_launches.csv $OUT/${TAG}_default_launches.md > /dev/null
rm -f $OUT/*.csv
ls -la $OUT
