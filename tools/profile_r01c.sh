#!/bin/bash
# Round-1 final refresh: bench lines of every configuration, the cfg5 launch list, ncu
# summaries of the fine sweep (cfg5), the SDIRK sweep (cfg4), the warp-specialised cluster
# coarse solve (cfg4), the level-2 sweep and the coarsest solve (cfg5).  Summaries are computed on the box and
# the .ncu-rep files dropped (gpurun copies back at most 64 MiB).
set -u
OUT=gpurun_out
python bench.py > $OUT/b_cfg5.json 2> $OUT/b_cfg5.err; echo "cfg5 rc=$?"
for c in cfg1_ideal cfg1_redisc cfg2 cfg3 cfg4 cfg4_literal; do
  python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/b_$c.json 2>> $OUT/b_other.err
  echo "$c rc=$?"
done
python bench.py --cycle F --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/b_cfg5_F.json 2>> $OUT/b_other.err
echo "cfg5 F rc=$?"
python bench.py --impl reference --steps 1 --warmup 0 > $OUT/b_reference.json 2>> $OUT/b_other.err
echo "reference rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
C4="python bench.py --config cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_r01c.csv $CMD > $OUT/ncu_launch_r01c.log 2>&1
echo "launch rc=$?"
python tools/launch_summary.py $OUT/launches_r01c.csv $OUT/launches_r01c_summary.json > $OUT/launches_r01c_summary.txt
prof() {  # name regex skip cmd...
  local name=$1 rx=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o $OUT/$name "$@" \
      > $OUT/ncu_$name.log 2>&1
  echo "$name rc=$?"
  python tools/ncu_summary.py $OUT/$name.ncu-rep > $OUT/${name}_ncu.json
  python tools/ncu_source_top.py $OUT/$name.ncu-rep 40 > $OUT/${name}_source_top.txt
  rm -f $OUT/$name.ncu-rep
}
prof fine_r01c rk_sweep_tma_kernel 1 $CMD
prof level2_r01c psi_level_kernel 0 $CMD
prof sdirk_r01c rk_sweep_kernel 2 $C4
prof coarse_tb_r01c psi_seq_cluster_tb_kernel 1 $C4
prof coarsest_r01c psi_coarse_kernel 0 $CMD
