#!/bin/bash
# compute-sanitizer over tools/sanitize.py, one case per process (each under its own
# timeout).  usage: tools/sanitize.sh racecheck|synccheck|memcheck [case ...]
tool=${1:-racecheck}; shift
cases=${@:-"tiles_vcycle cluster_tb cluster_ca cluster_plain seq_periodic whole_rows sdirk rk_coarse_ideal rk_coarse_redisc"}
mkdir -p gpurun_out
for c in $cases; do
  echo "=== $tool $c"
  timeout ${SAN_TIMEOUT:-600} compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py $c 2>&1 | tail -25
  echo "exit ${PIPESTATUS[0]}"
done
