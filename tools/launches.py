"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list.

Steps are counted as the launch count of the once-per-step dispatch kernel
(k_dispatch), so kernels launched twice per step (the two compensation GEMMs)
contribute both launches to the per-step total."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
agg = collections.OrderedDict()
for d in data:
    if "xg::" not in d["Kernel Name"] and "k_" not in d["Kernel Name"]:
        continue  # library kernels of the bench's reference points (cuBLASLt, torch RNG)
    agg.setdefault(d["Kernel Name"].split("(")[0][-48:], []).append(float(d["Metric Value"]))
steps = next((len(v) for n, v in agg.items() if "k_dispatch" in n), None) or min(len(v) for v in agg.values())
tot = 0.0
for n, v in agg.items():
    if "generate" in n:
        continue
    per = sum(v) / len(v)
    step = sum(v) / steps
    tot += step
    print(f"{len(v):4d} x {per / 1e3:9.1f} us  ({step / 1e3:7.1f} us/step)  {n}")
print(f"steps: {steps}; sum of kernel time per step: {tot / 1e3:.1f} us")
