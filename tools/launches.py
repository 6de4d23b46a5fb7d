"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
agg = collections.OrderedDict()
for d in data:
    agg.setdefault(d["Kernel Name"].split("(")[0][-48:], []).append(float(d["Metric Value"]))
tot = 0.0
for n, v in agg.items():
    if "generate" in n:
        continue
    per = sum(v) / len(v)
    tot += per
    print(f"{len(v):4d} x {per / 1e3:9.1f} us  {n}")
print(f"sum of per-step kernel means: {tot / 1e3:.1f} us")
