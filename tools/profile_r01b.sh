#!/bin/bash
# Round-1 refresh: bench lines of every configuration, cfg5 launch list, ncu of the fine
# sweep (cfg5) and of the SDIRK sweep (cfg4).  Run from the repo root under gpurun.
set -u
OUT=gpurun_out
python bench.py > $OUT/b_cfg5.json 2> $OUT/b_cfg5.err; echo "cfg5 rc=$?"
for c in cfg1_ideal cfg1_redisc cfg2 cfg3 cfg4 cfg4_literal; do
  python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/b_$c.json 2>> $OUT/b_other.err
  echo "$c rc=$?"
done
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_r01b.csv $CMD > $OUT/ncu_launch_r01b.log 2>&1
echo "launch rc=$?"
ncu --set full --clock-control none --import-source on -k regex:rk_sweep_tma_kernel -s 1 -c 1 \
    -o $OUT/fine_r01b $CMD > $OUT/ncu_fine_r01b.log 2>&1
echo "fine rc=$?"
ncu --set full --clock-control none --import-source on -k regex:rk_sweep_kernel -s 2 -c 1 \
    -o $OUT/sdirk_r01b python bench.py --config cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
    > $OUT/ncu_sdirk_r01b.log 2>&1
echo "sdirk rc=$?"
python tools/launch_summary.py $OUT/launches_r01b.csv $OUT/launches_r01b_summary.json > $OUT/launches_r01b_summary.txt
python tools/ncu_summary.py $OUT/fine_r01b.ncu-rep > $OUT/fine_r01b_ncu.json
python tools/ncu_source_top.py $OUT/fine_r01b.ncu-rep 40 > $OUT/fine_r01b_source_top.txt
python tools/ncu_summary.py $OUT/sdirk_r01b.ncu-rep > $OUT/sdirk_r01b_ncu.json
python tools/ncu_source_top.py $OUT/sdirk_r01b.ncu-rep 40 > $OUT/sdirk_r01b_source_top.txt
rm -f $OUT/*.ncu-rep
