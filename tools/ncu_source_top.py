"""Top SASS instructions by warp-stall samples with their dominant stall reasons.
usage: python tools/ncu_source_top.py <report.ncu-rep> [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, rows = r[1], r[2:]
i_s = h.index("Warp Stall Sampling (All Samples)")
i_src, i_ex = h.index("Source"), h.index("Instructions Executed")
st = [k for k, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


tot = sum(f(x[i_s]) for x in rows)
print("total samples", tot)
for k, x in enumerate(rows):
    x.append(k)
for x in sorted(rows, key=lambda x: -f(x[i_s]))[:n]:
    reasons = sorted(((f(x[k]), h[k][6:]) for k in st), reverse=True)[:2]
    rs = " ".join(f"{nm}={v:.0f}" for v, nm in reasons if v > 0)
    print(f"#{x[-1]:4d} {f(x[i_s]) / tot * 100:5.1f}% {x[i_ex]:>7} {x[i_src][:60]:60s} {rs}")
