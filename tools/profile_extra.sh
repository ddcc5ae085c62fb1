# ncu of the cfg5 level-2 interpolation (8th psi_level_kernel launch of a solve) and of the
# check sweep (7th rk_sweep_tma_kernel launch), summarised on the box.
OUT=gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > /dev/null 2>&1 || exit 1
prof() {
  local name=$1 rx=$2 skip=$3
  ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o $OUT/$name $CMD \
      > $OUT/ncu_$name.log 2>&1
  echo "$name rc=$?"
  python tools/ncu_summary.py $OUT/$name.ncu-rep > $OUT/${name}_ncu.json
  python tools/ncu_source_top.py $OUT/$name.ncu-rep 30 > $OUT/${name}_source_top.txt
  rm -f $OUT/$name.ncu-rep
}
# prof interp2_r01c psi_level_kernel 7
# prof check_r01c rk_sweep_tma_kernel 6
prof coarsest_r01c psi_coarse_kernel 0
