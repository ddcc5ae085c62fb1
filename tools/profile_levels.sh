#!/bin/bash
set -u
TAG=${1:-r01}
OUT=gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > $OUT/prof_plain_$TAG.json 2> $OUT/prof_plain_$TAG.err || { echo "plain run failed"; exit 1; }
# level-2 sweep = 1st psi_level launch of a V-cycle, level-2 interp = 8th
ncu --set full --clock-control none --import-source on -k regex:psi_level_kernel -s 8 -c 8 \
    -o $OUT/levels_$TAG $CMD > $OUT/ncu_levels_$TAG.log 2>&1
echo "levels rc=$?"
