# A/B two builds of the library on one box: libmgrit.so (new) vs libmgrit_old.so (old)
cp paper_1910_03726_b200/libmgrit.so /tmp/new.so
for rep in 1 2 3; do for v in old new; do
  cp /tmp/$v.so paper_1910_03726_b200/libmgrit.so 2>/dev/null || cp paper_1910_03726_b200/libmgrit_old.so paper_1910_03726_b200/libmgrit.so
  [ $v = old ] && cp paper_1910_03726_b200/libmgrit_old.so paper_1910_03726_b200/libmgrit.so
  touch paper_1910_03726_b200/libmgrit.so
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);s=d['kernel_time_share'];print('$v', d['ms_per_step'], 'fine', d['roofline']['avg_launch_ms'], 'coarse', d['coarse_solve']['ns_per_step'])"
done; done
cp /tmp/new.so paper_1910_03726_b200/libmgrit.so; touch paper_1910_03726_b200/libmgrit.so
timeout 600 python -m pytest tests -m gpu -x -q -k "cfg5 or vcycle or hierarch or fcycle or deterministic or sdirk_multilevel" 2>&1 | tail -1
