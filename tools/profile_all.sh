#!/bin/bash
# Run on the GPU box (gpurun): bench lines of every config, the ncu launch list of the default
# command and one `ncu --set full` capture per key kernel, summarised by tools/ncu_summary.py.
# Outputs land in gpurun_out/prof/ (copy what should be judged into profiles/).
#   bash tools/profile_all.sh <tag>
set -u
TAG=${1:-r2}
OUT=gpurun_out/prof
mkdir -p $OUT
NCU="ncu --clock-control none"

# 1. bench lines (never under a profiler)
for c in 0 1 2; do
  python bench.py --config $c > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
done
python bench.py --config 4 --phase steps > $OUT/bench_c4s.json 2> $OUT/bench_c4s.err

# 2. launch list of the default command
$NCU --metrics gpu__time_duration.sum -c 6000 --csv --log-file $OUT/${TAG}_default_launches.csv \
  python bench.py --steps 2 --warmup 3 > $OUT/ncu_default.log 2>&1
python tools/ncu_summary.py launches $OUT/${TAG}_default_launches.csv $OUT/${TAG}_default_launches.md > /dev/null

# 3. full captures, one kernel family per call
cap() {  # name config kernel-regex count [extra bench args]
  local name=$1 cfg=$2 rx=$3 cnt=$4; shift 4
  $NCU --set full --import-source on -k "regex:$rx" --launch-skip 2 -c $cnt -f -o $OUT/${TAG}_$name \
    python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline "$@" > $OUT/ncu_$name.log 2>&1
  python tools/ncu_summary.py report $OUT/${TAG}_$name.ncu-rep $OUT/${TAG}_${name}_full > /dev/null 2>> $OUT/ncu_$name.log
  keep_source $name
}
# gpurun copies back <= 64 MiB: keep the summaries, the per-line source page (gzip) of the
# kernels being tuned, and drop the reports themselves
keep_source() {
  case $1 in
    c4_rbf|c4_knn|c1_rbf|c3_trisolve)
      ncu -i $OUT/${TAG}_$1.ncu-rep --page source --csv 2>/dev/null | gzip -9 > $OUT/${TAG}_$1_source.csv.gz ;;
  esac
  rm -f $OUT/${TAG}_$1.ncu-rep
}
cap c0_mon 0 'mon_weights_kernel' 1
cap c0_apply 0 'apply_ell_kernel' 1
cap c1_rbf 1 'rbf_static_kernel|rbf_ns_kernel' 1
cap c1_knn 1 'knn_' 2
cap c1_apply 1 'apply_ell_kernel' 1
cap c2_rbf 2 'rbf_static_kernel|rbf_ns_kernel|mon_weights_kernel' 2
cap c2_apply 2 'apply_ell_kernel' 1
cap c4_rbf 4 'rbf_ns_kernel' 1 --no-steps
cap c4_knn 4 'knn_' 2 --no-steps
cap c4_mon 4 'mon_weights_kernel|mon_stencil_kernel' 2 --no-steps
cap c4_apply 4 'apply_ell_kernel' 1 --no-steps
# config-3 step: ncu does not descend into the conditional graph node, so the dev-only eager mode
cap3() {  # name kernel-regex count
  HN_PRESSURE_EAGER=1 $NCU --set full --import-source on -k "regex:$2" --launch-skip 4 -c $3 -f -o $OUT/${TAG}_$1 \
    python tools/prof_step_eager.py 4 > $OUT/ncu_$1.log 2>&1
  python tools/ncu_summary.py report $OUT/${TAG}_$1.ncu-rep $OUT/${TAG}_${1}_full > /dev/null 2>> $OUT/ncu_$1.log
  keep_source $1
}
cap3 c3_explicit 'momentum_fused_kernel|div_rhs_fused_kernel|correct_temp_fused_kernel|temperature_bc_kernel' 4
cap3 c3_trisolve 'sptrsv_super_kernel' 2
HN_PRESSURE_EAGER=1 $NCU --metrics gpu__time_duration.sum -c 4000 --csv --log-file $OUT/${TAG}_c3_step_launches.csv \
  python tools/prof_step_eager.py 6 > $OUT/ncu_c3_step.log 2>&1
python tools/ncu_summary.py launches $OUT/${TAG}_c3_step_launches.csv $OUT/${TAG}_c3_step_launches.md > /dev/null
ls -la $OUT
