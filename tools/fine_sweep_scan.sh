#!/bin/bash
# Fine-sweep configuration scan (bench cfg5, fine_sweep avg launch time per config).
for cfg in ${CFGS:-"256,11" "128,15" "128,15,2"}; do
  python bench.py --opt fine_tile=$cfg --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', 'ms/solve', d['ms_per_step'], 'K', d['config']['iterations'], 'fine avg ms', r['avg_launch_ms'], 'frac', r['frac'], d['kernel_time_share'])"
done
