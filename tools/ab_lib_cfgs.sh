# A/B two builds (libmgrit.so new vs libmgrit_old.so) on the two-level configurations
cp paper_1910_03726_b200/libmgrit.so /tmp/new.so
cp paper_1910_03726_b200/libmgrit_old.so /tmp/old.so
for rep in 1 2; do for v in old new; do
  cp /tmp/$v.so paper_1910_03726_b200/libmgrit.so; touch paper_1910_03726_b200/libmgrit.so
  for c in cfg1_redisc cfg2 cfg3 cfg4; do
    python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$v', '$c', d['ms_per_step'], 'fine', d['roofline']['avg_launch_ms'])"
  done
done; done
cp /tmp/new.so paper_1910_03726_b200/libmgrit.so; touch paper_1910_03726_b200/libmgrit.so
