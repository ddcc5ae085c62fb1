# Coarse-solve configuration scan (tools/coarse_probe.py): cluster split x s-step depth.
for cfgs in "16,128,2" "16,64,4"; do for S in 3 4 6 8; do
  timeout 120 python tools/coarse_probe.py cfg4 3 seq_cluster=$cfgs seq_s=$S 2>&1 | tail -1 | sed "s/^/$cfgs S=$S /"
done; done
for cfgs in "16,128,2" "16,64,4"; do for S in 4 6 8 10; do
  timeout 120 python tools/coarse_probe.py cfg3 3 seq_cluster=$cfgs seq_s=$S 2>&1 | tail -1 | sed "s/^/$cfgs S=$S /"
done; done
for S in 6 8 12 16; do
  timeout 120 python tools/coarse_probe.py cfg2 3 seq_cluster=16,32,2 seq_s=$S 2>&1 | tail -1 | sed "s/^/16,32,2 S=$S /"
done
