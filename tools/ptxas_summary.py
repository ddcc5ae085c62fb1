"""Summarise ptxas -v output: kernel, registers, spill bytes, smem."""
import re, subprocess, sys
log = open(sys.argv[1]).read().splitlines()
cur = None
rows = []
for line in log:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        cur["spill"] = int(m.group(1)) + int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur["regs"] = int(m.group(1))
names = [r["name"] for r in rows]
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
for r, d in zip(rows, dem):
    d = re.sub(r"mg::Scheme<(\d+), (\d+), (\d+), \d+ul, \d+u, false>", r"S\1L\2R\3", d)
    d = d.replace("void mg::", "").replace("(mg::SweepArgs)", "").replace("(mg::CoarseArgs)", "").replace("(mg::PsiSweepArgs)", "").replace("(mg::RKCoarseArgs)","")
    print(f"{r.get('regs','?'):>4} regs  spill {r.get('spill',0):>5}  {d}")
