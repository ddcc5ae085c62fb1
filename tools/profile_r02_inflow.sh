#!/bin/bash
# ncu --set full summaries of the inflow/outflow kernels added after tools/profile_r02.sh: the
# truncated cluster chain (inflow_erk3, serial iteration: ncu replays kernels one at a time) and
# the truncated level kernel (inflow_erk3_ml).
set -u
OUT=gpurun_out
CI="python bench.py --config inflow_erk3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --opt overlap=0 --opt graph=0"
CM="python bench.py --config inflow_erk3_ml --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --opt graph=0"
prof() {
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o $OUT/$name "$@" \
      > $OUT/ncu_$name.log 2>&1
  echo "$name rc=$?"
  python tools/ncu_summary.py $OUT/$name.ncu-rep > $OUT/${name}_ncu.json
  python tools/ncu_source_top.py $OUT/$name.ncu-rep 40 > $OUT/${name}_source_top.txt
  rm -f $OUT/$name.ncu-rep
}
prof r02_inflow_chain_tb psi_seq_cluster_tb_kernel 1 $CI
prof r02_inflow_tpsi_level tpsi_level_kernel 2 $CM
