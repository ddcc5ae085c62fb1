#!/bin/bash
set -u
TAG=${1:-r01}
OUT=gpurun_out
CMD="python bench.py --config ${CFG:-cfg2} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > $OUT/prof_plain_$TAG.json 2> $OUT/prof_plain_$TAG.err || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-psi_coarse_kernel} -s 2 -c 1 \
    -o $OUT/coarse_$TAG $CMD > $OUT/ncu_coarse_$TAG.log 2>&1
echo "coarse rc=$?"
