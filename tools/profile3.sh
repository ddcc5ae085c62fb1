#!/bin/bash
set -u
TAG=${1:-r01}
OUT=gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > $OUT/prof_plain_$TAG.json 2> $OUT/prof_plain_$TAG.err || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1
echo "launch rc=$?"
ncu --set full --clock-control none --import-source on -k regex:rk_sweep_tma_kernel -s 1 -c 1 \
    -o $OUT/fine_tma_$TAG $CMD > $OUT/ncu_fine_$TAG.log 2>&1
echo "fine rc=$?"
ncu --set full --clock-control none --import-source on -k regex:psi_level_kernel -s 4 -c 1 \
    -o $OUT/interp_$TAG $CMD > $OUT/ncu_interp_$TAG.log 2>&1
echo "interp rc=$?"
