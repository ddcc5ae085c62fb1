#!/bin/bash
# A/B of fine-sweep tiles on cfg5 within one box: default then each --opt fine_tile.
for cfg in default ${CFGS:-"32,15" "32,23" "32,31"}; do
  if [ "$cfg" = default ]; then o=""; else o="--opt fine_tile=$cfg"; fi
  python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $o 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', 'ms/solve', d['ms_per_step'], 'K', d['config']['iterations'], 'fine avg ms', r['avg_launch_ms'], 'frac', r['frac'], 'clk', d['clocks']['sm_mhz'])"
done
