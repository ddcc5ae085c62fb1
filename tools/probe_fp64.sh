#!/bin/bash
# FP64 DFMA peak probe with an nvidia-smi clock record (the roofline denominator of the
# fine sweep).  Writes profiles/r02_fp64_probe.txt (+ .json: the summary).
set -e
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probe_fp64.cu -o tools/probe_fp64
mkdir -p profiles
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active \
  --format=csv -lms 100 > /tmp/probe_clocks.csv & SMI=$!
sleep 0.5
./tools/probe_fp64 > /tmp/probe_out.txt
sleep 0.3; kill $SMI || true
{ echo "# tools/probe_fp64 (DFMA chains, ILP 8) on $(nvidia-smi --query-gpu=name --format=csv,noheader)";
  cat /tmp/probe_out.txt; echo "# nvidia-smi samples during the run"; cat /tmp/probe_clocks.csv; } \
  > profiles/r02_fp64_probe.txt
python - <<'PY'
import json, statistics
rows = [l.split(",") for l in open("/tmp/probe_clocks.csv").read().splitlines()[1:] if l.strip()]
sm = [float(r[1].split()[0]) for r in rows if len(r) > 2]
load = [v for v in sm if v > 600]
summ = json.loads([l for l in open("/tmp/probe_out.txt") if l.startswith("{")][0])
summ["sm_mhz_median_under_load"] = statistics.median(load) if load else None
summ["sm_max_mhz"] = float(rows[0][2].split()[0]) if rows else None
json.dump(summ, open("profiles/r02_fp64_probe.json", "w"), indent=1)
print(summ)
PY
