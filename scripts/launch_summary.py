"""Summarise an ncu launch list (gpu__time_duration.sum per launch): our kernels, their share."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
ours = [(r[ki], float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "ns" else 1.0)) for r in rows[1:]
        if "earl::" in r[ki]]
tot = sum(t for _, t in ours)
agg = defaultdict(list)
for k, t in ours:
    agg[k.split("(")[0]].append(t)
print(f"launches of libearl_dispatch.so kernels: {len(ours)}  (ncu: cold-cache, serialised)")
print(f"{'kernel':70s} {'n':>4s} {'avg us':>10s} {'share':>7s}")
for k, ts in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:70]:70s} {len(ts):4d} {sum(ts)/len(ts):10.2f} {sum(ts)/tot*100:6.2f}%")
