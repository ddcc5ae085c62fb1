#!/bin/bash
# Usage (under gpurun): bash tools/profile.sh <tag>
# 1) plain bench run (must exit 0), 2) ncu launch list, 3) ncu --set full of the fine sweep.
set -u
TAG=${1:-r01}
OUT=gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > $OUT/prof_plain_$TAG.json 2> $OUT/prof_plain_$TAG.err || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:rk_sweep_kernel -s 1 -c 1 \
    -o $OUT/fine_sweep_$TAG $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
