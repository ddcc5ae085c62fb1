#!/bin/bash
# ncu --set full of the two big V-cycle level kernels of cfg5 (level-2 sweep: first
# psi_level_kernel launch; level-2 -> level-1 interpolation: eighth), summarised on the box.
set -u
TAG=${1:-r01}
OUT=gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
$CMD > $OUT/prof_plain_$TAG.json 2> $OUT/prof_plain_$TAG.err || { echo "plain run failed"; exit 1; }
for spec in "sweep 0" "interp 7"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:psi_level_kernel -s $2 -c 1 \
      -o $OUT/lvl_${1}_$TAG $CMD > $OUT/ncu_lvl_${1}_$TAG.log 2>&1
  echo "$1 rc=$?"
  python tools/ncu_summary.py $OUT/lvl_${1}_$TAG.ncu-rep --json $OUT/lvl_${1}_${TAG}_summary.json > /dev/null
  python tools/ncu_source_top.py $OUT/lvl_${1}_$TAG.ncu-rep 30 > $OUT/lvl_${1}_${TAG}_source_top.txt
done
