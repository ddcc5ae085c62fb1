#!/bin/bash
# Round-2 refresh: the bench line (cfg5) and the reference arm, the other configurations and
# the inflow/outflow cases, the cfg5 launch list, and ncu --set full summaries of the fine
# sweep (cfg5), the SDIRK sweep and the cluster chain (cfg4), the inflow/outflow sweep and the
# truncated-Psi chain (inflow_erk3).  ncu replays kernels one at a time, so the two-level
# commands run with --opt overlap=0 (a speculative chain waits for sweeps that a serialised
# run never starts).  Summaries are computed on the box, the .ncu-rep files dropped.
set -u
OUT=gpurun_out
python bench.py > $OUT/bench_r02.json 2> $OUT/bench_r02.err; echo "cfg5 rc=$?"
python bench.py --impl reference --steps 1 --warmup 0 > $OUT/bench_r02_reference.json 2>> $OUT/b_other.err
echo "reference rc=$?"
for c in cfg1_ideal cfg1_redisc cfg2 cfg3 cfg4 cfg4_literal inflow_erk3 inflow_erk3_ml; do
  python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_r02_$c.json 2>> $OUT/b_other.err
  echo "$c rc=$?"
done
for c in cfg2 cfg3 cfg4; do
  python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --opt overlap=0 --opt graph=0 \
      > $OUT/bench_r02_${c}_serial.json 2>> $OUT/b_other.err
  echo "$c serial rc=$?"
done
python bench.py --cycle F --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_r02_cfg5_fcycle.json 2>> $OUT/b_other.err
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
C4="python bench.py --config cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --opt overlap=0 --opt graph=0"
CI="python bench.py --config inflow_erk3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/r02_launches.csv $CMD > $OUT/ncu_launch_r02.log 2>&1
echo "launch rc=$?"
python tools/launch_summary.py $OUT/r02_launches.csv $OUT/r02_launches_summary.json > $OUT/r02_launches_summary.txt
prof() {  # name regex skip cmd...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o $OUT/$name "$@" \
      > $OUT/ncu_$name.log 2>&1
  echo "$name rc=$?"
  python tools/ncu_summary.py $OUT/$name.ncu-rep > $OUT/${name}_ncu.json
  python tools/ncu_source_top.py $OUT/$name.ncu-rep 40 > $OUT/${name}_source_top.txt
  rm -f $OUT/$name.ncu-rep
}
prof r02_fine_sweep rk_sweep_tma_kernel 1 $CMD
prof r02_sdirk_sweep_cfg4 rk_sweep_kernel 2 $C4
prof r02_coarse_tb_cfg4 psi_seq_cluster_tb_kernel 1 $C4
prof r02_inflow_sweep rk_sweep_kernel 2 $CI
prof r02_inflow_tpsi_seq tpsi_seq_kernel 1 $CI
