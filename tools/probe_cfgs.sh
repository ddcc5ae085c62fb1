# Coarse-solve configuration scan (tools/coarse_probe.py): cluster split x s-step depth.
for cfgs in "16,128,2" "16,64,4"; do for S in 3 4 6 8; do
  MGRIT_SEQ_CLUSTER=$cfgs MGRIT_SEQ_S=$S timeout 120 python tools/coarse_probe.py cfg4 3 2>&1 | tail -1 | sed "s/^/$cfgs S=$S /"
done; done
for cfgs in "16,128,2" "16,64,4"; do for S in 4 6 8 10; do
  MGRIT_SEQ_CLUSTER=$cfgs MGRIT_SEQ_S=$S timeout 120 python tools/coarse_probe.py cfg3 3 2>&1 | tail -1 | sed "s/^/$cfgs S=$S /"
done; done
for S in 6 8 12 16; do
  MGRIT_SEQ_CLUSTER=16,32,2 MGRIT_SEQ_S=$S timeout 120 python tools/coarse_probe.py cfg2 3 2>&1 | tail -1 | sed "s/^/16,32,2 S=$S /"
done
