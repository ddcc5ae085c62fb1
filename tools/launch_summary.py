"""Summarise an ncu launch list (gpu__time_duration per launch): per-kernel totals and shares."""
import csv, collections, re, sys, json
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]; data = rows[hdr_i + 1:]
ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit'); gi = hdr.index('Grid Size')
agg = collections.OrderedDict(); tot = 0.0
for r in data:
    name = re.sub(r'\(.*', '', r[ki]); name = re.sub(r'mg::Scheme<[^>]*>', 'S', name).replace('void mg::', '').replace('mg::', '')
    key = f"{name} grid{r[gi]}"
    v = float(r[vi].replace(',', '')) * {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3}.get(r[ui], 1)
    agg.setdefault(key, [0, 0.0]); agg[key][0] += 1; agg[key][1] += v; tot += v
out = [{"kernel": k, "launches": n, "total_us": round(t, 1), "avg_us": round(t / n, 1), "share": round(t / tot, 4)}
       for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]
print(f"{'share':>6} {'total_ms':>9} {'n':>4} {'avg_us':>9}  kernel")
for o in out:
    print(f"{100*o['share']:5.1f}% {o['total_us']/1e3:9.3f} {o['launches']:4d} {o['avg_us']:9.1f}  {o['kernel']}")
print("total ms", round(tot / 1e3, 3), "launches", len(data))
if len(sys.argv) > 2:
    json.dump({"total_ms": tot / 1e3, "launches": len(data), "kernels": out}, open(sys.argv[2], "w"), indent=1)
