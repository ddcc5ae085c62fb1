python paper_1910_03726_b200/build.py >/dev/null
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 600 gpurun_out/bench_default.json
for c in cfg1_ideal cfg1_redisc cfg2 cfg3 cfg4 cfg4_literal; do timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_$c.json; done
bash tools/profile3.sh r01k
CFG=cfg3 KREGEX=psi_seq_cluster bash tools/profile_coarse.sh r01k3
CFG=cfg4 KREGEX=psi_seq_cluster bash tools/profile_coarse.sh r01k4
for r in fine_tma_r01k interp_r01k coarse_r01k3 coarse_r01k4; do python tools/ncu_summary.py gpurun_out/$r.ncu-rep --json gpurun_out/${r}_summary.json > /dev/null; python tools/ncu_source_top.py gpurun_out/$r.ncu-rep 30 > gpurun_out/${r}_source_top.txt; done
python tools/launch_summary.py gpurun_out/launches_r01k.csv > gpurun_out/launches_r01k_summary.txt
rm -f gpurun_out/fine_tma_r01k.ncu-rep gpurun_out/interp_r01k.ncu-rep
du -sh gpurun_out
