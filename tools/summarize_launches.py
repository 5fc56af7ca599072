"""Summarise an ncu --metrics gpu__time_duration.sum CSV into per-kernel shares."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
i_name, i_val, i_metric = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= i_val or r[i_metric] != "gpu__time_duration.sum":
        continue
    name = r[i_name].split("(")[0].replace("void ", "")
    v = float(r[i_val].replace(",", ""))
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v for _, v in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {c:8d} {v/1e6:10.3f} {100*v/tot:6.1f}%")
print(f"{'TOTAL':60s} {sum(c for c,_ in agg.values()):8d} {tot/1e6:10.3f}")
