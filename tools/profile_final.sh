#!/bin/bash
# Final-code refresh of the captures whose kernels changed late in the round (GPU box):
# the 2D RBF sweep kernel (config 1) and the fused explicit kernels (config 3).
#   bash tools/profile_final.sh <tag>
set -u
TAG=${1:-r2}
OUT=gpurun_out/prof
mkdir -p $OUT
NCU="ncu --clock-control none"
$NCU --set full -k "regex:rbf_static_kernel" --launch-skip 2 -c 1 -f -o $OUT/${TAG}_c1_rbf \
  python bench.py --config 1 --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_c1_rbf.log 2>&1
python tools/ncu_summary.py report $OUT/${TAG}_c1_rbf.ncu-rep $OUT/${TAG}_c1_rbf_full > /dev/null 2>> $OUT/ncu_c1_rbf.log
HN_PRESSURE_EAGER=1 $NCU --set full -k "regex:momentum_fused_kernel|div_rhs_fused_kernel|correct_temp_fused_kernel|temperature_bc_kernel" \
  --launch-skip 4 -c 4 -f -o $OUT/${TAG}_c3_explicit python tools/prof_step_eager.py 4 > $OUT/ncu_c3_explicit.log 2>&1
python tools/ncu_summary.py report $OUT/${TAG}_c3_explicit.ncu-rep $OUT/${TAG}_c3_explicit_full > /dev/null 2>> $OUT/ncu_c3_explicit.log
rm -f $OUT/*.ncu-rep
