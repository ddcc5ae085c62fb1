# ncu of the all-row residual of the guess (K2 standalone, rk_residual_tma_kernel), cfg5.
OUT=gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rk_residual_tma_kernel -s 0 -c 1 \
    -o $OUT/residual_r01c $CMD > $OUT/ncu_residual.log 2>&1
python tools/ncu_summary.py $OUT/residual_r01c.ncu-rep > $OUT/residual_r01c_ncu.json
python tools/ncu_source_top.py $OUT/residual_r01c.ncu-rep 30 > $OUT/residual_r01c_source_top.txt
rm -f $OUT/*.ncu-rep
