"""Per-kernel mean time and DRAM bytes from an ncu --csv launch list taken with
several --metrics (e.g. gpu__time_duration.sum,dram__bytes_read.sum)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
d = collections.defaultdict(lambda: collections.defaultdict(list))
order = []
for r in rows[start + 1:]:
    x = dict(zip(h, r))
    k = x["Kernel Name"][:48]
    if k not in d:
        order.append(k)
    d[k][x["Metric Name"]].append(float(x["Metric Value"].replace(",", "")))
for k in order:
    v = d[k]
    t = v.get("gpu__time_duration.sum", [])
    b = v.get("dram__bytes_read.sum", [])
    w = v.get("dram__bytes_write.sum", [])
    line = f"{k:50s} n={len(t):3d} t={sum(t) / len(t) / 1000 if t else 0:9.1f} us"
    if b:
        line += f" rd={sum(b) / len(b) / 1e6:8.1f} MB"
    if w:
        line += f" wr={sum(w) / len(w) / 1e6:8.1f} MB"
    print(line)
