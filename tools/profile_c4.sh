#!/bin/bash
# Config-4 weights profile of the final code (GPU box): full captures of the RBF solve and the kNN
# kernel (summaries only) and the launch list of the weights-only command.
#   bash tools/profile_c4.sh <tag>
set -u
TAG=${1:-r2}
OUT=gpurun_out/prof
mkdir -p $OUT
NCU="ncu --clock-control none"
for spec in "c4_rbf:rbf_ns_kernel:1" "c4_knn:knn_warp_kernel:1"; do
  IFS=: read name rx cnt <<< "$spec"
  $NCU --set full -k "regex:$rx" --launch-skip 2 -c $cnt -f -o $OUT/${TAG}_$name \
    python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-steps > $OUT/ncu_$name.log 2>&1
  python tools/ncu_summary.py report $OUT/${TAG}_$name.ncu-rep $OUT/${TAG}_${name}_full > /dev/null 2>> $OUT/ncu_$name.log
  rm -f $OUT/${TAG}_$name.ncu-rep
done
$NCU --metrics gpu__time_duration.sum -c 3000 --csv --log-file $OUT/${TAG}_c4_launches.csv \
  python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-steps > $OUT/ncu_c4.log 2>&1
python tools/ncu_summary.py launches $OUT/${TAG}_c4_launches.csv $OUT/${TAG}_c4_launches.md > /dev/null
rm -f $OUT/*.csv
