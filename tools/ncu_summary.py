"""Summarise an ncu report (raw page): per kernel duration (ms), DRAM bytes (GB), pipe
utilisations and the top stall reasons.  Units are normalised from ncu's unit row.

usage: python tools/ncu_summary.py <report.ncu-rep> [--json out.json]
"""
import csv
import json
import subprocess
import sys

TIME = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
        "second": 1e3, "s": 1e3}
BYTES = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    res = []
    for v in r[2:]:
        d = dict(zip(h, v))
        u = dict(zip(h, units))

        def f(k, scale=None):
            try:
                x = float(d.get(k, "nan").replace(",", ""))
            except ValueError:
                return None
            if scale is not None:
                x *= scale.get(u.get(k, ""), 1.0)
            return x

        stalls = {}
        for name, val in d.items():
            if "average_warps_issue_stalled" in name and name.endswith("_per_issue_active.ratio"):
                try:
                    stalls[name.split("stalled_")[1].replace("_per_issue_active.ratio", "")] = float(val)
                except ValueError:
                    pass
        rd = f("dram__bytes_read.sum", BYTES)
        wr = f("dram__bytes_write.sum", BYTES)
        res.append({
            "kernel": d.get("Kernel Name", "")[:100], "grid": d.get("Grid Size"),
            "block": d.get("Block Size"),
            "duration_ms": f("gpu__time_duration.sum", TIME),
            "dram_read_GB": rd, "dram_write_GB": wr,
            "dram_bytes_per_launch": None if rd is None or wr is None else (rd + wr) * 1e9,
            "dram_throughput_pct": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "sm_throughput_pct": f("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "registers": f("launch__registers_per_thread"),
            "stalls_top": dict(sorted(stalls.items(), key=lambda x: -x[1])[:7]),
        })
    return res


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
    print(json.dumps(res, indent=1))
