"""Summarise an ncu report: per kernel duration, throughput, DRAM bytes, DFMA rate, stalls."""
import csv, subprocess, sys, json
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
res = []
for v in r[2:]:
    d = dict(zip(h, v))
    def f(k):
        try: return float(d.get(k, "nan").replace(",", ""))
        except: return None
    stalls = {}
    for name, val in d.items():
        if 'average_warps_issue_stalled' in name and name.endswith('_per_issue_active.ratio'):
            try: stalls[name.split('stalled_')[1].replace('_per_issue_active.ratio','')] = float(val)
            except: pass
    top = dict(sorted(stalls.items(), key=lambda x: -x[1])[:7])
    k = {"kernel": d.get("Kernel Name", "")[:90], "grid": d.get("Grid Size"), "block": d.get("Block Size"),
         "duration_ms": f("gpu__time_duration.sum"),
         "sm_throughput_pct": f("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
         "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
         "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
         "dram_read_GB": f("dram__bytes_read.sum"), "dram_write_GB": f("dram__bytes_write.sum"),
         "dram_throughput_pct": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
         "dfma_per_cycle_per_smsp": f("smsp__sass_thread_inst_executed_op_dfma_pred_on.avg.per_cycle_elapsed"),
         "fp64_pipe_pct_of_peak": None,
         "registers": f("launch__registers_per_thread"), "stalls_top": top}
    if k["dfma_per_cycle_per_smsp"] is not None:
        k["fp64_pipe_pct_of_peak"] = 100 * k["dfma_per_cycle_per_smsp"] / 16.0
    res.append(k)
print(json.dumps(res, indent=1))
