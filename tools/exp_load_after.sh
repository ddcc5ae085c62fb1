#!/bin/bash
# Experiment: position of the thread-0 prefetch in the fine sweep (MGRIT_LOAD_AFTER).
set -u
for la in 1 2 3; do
  MGRIT_LOAD_AFTER=$la python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_la$la.json 2>>gpurun_out/exp.err
  echo "la=$la rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:rk_sweep_tma_kernel -s 1 -c 1 \
    -o gpurun_out/fine_src python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_fine.log 2>&1
echo "ncu rc=$?"
