# ncu of the cfg5 V-cycle level-2 sweep (first psi_level_kernel launch) and interpolation.
OUT=gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:psi_level_kernel -s 0 -c 1 \
    -o $OUT/lev2_sweep $CMD > $OUT/ncu_lev2.log 2>&1
python tools/ncu_summary.py $OUT/lev2_sweep.ncu-rep > $OUT/lev2_sweep_ncu.json
python tools/ncu_source_top.py $OUT/lev2_sweep.ncu-rep 30 > $OUT/lev2_sweep_source_top.txt
rm -f $OUT/*.ncu-rep
