"""Top SASS instructions by warp-stall samples from an .ncu-rep (source page),
per kernel: python tools/ncu_sass_hot.py rep.ncu-rep [kernel-substring] [N]"""
import csv, io, subprocess, sys

path = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
sections, cur = [], None
for row in csv.reader(io.StringIO(out)):
    if row and row[0] == "Kernel Name":
        cur = [row[1], None, []]
        sections.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = row
    elif cur is not None:
        cur[2].append(row)
for name, hdr, rows in sections:
    if want not in name:
        continue
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_n = hdr.index("Warp Stall Sampling (Not-issued Samples)")
    tot = sum(float(r[i_s] or 0) for r in rows)
    print(f"== {name}  total samples {tot:.0f}")
    idx = sorted(range(len(rows)), key=lambda k: -float(rows[k][i_s] or 0))[:topn]
    for k in sorted(idx):
        r = rows[k]
        print(f"{k:5d} {r[0]:>6} {float(r[i_s] or 0) / tot * 100:5.1f}% ns {float(r[i_n] or 0) / tot * 100:5.1f}%  {r[1][:90]}")
