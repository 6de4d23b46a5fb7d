"""Per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per
launch from an `ncu --set full` capture, written as JSON for bench.py's
roofline.traffic field.  Usage: python tools/ncu_traffic.py rep.ncu-rep out.json"""
import csv
import io
import json
import subprocess
import sys


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    agg = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0]
        b = sum(float(d[m].replace(",", "")) * scale.get(units[m], 1) for m in
                ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        agg.setdefault(name, []).append(b)
    res = {k: {"bytes_per_launch": sum(v) / len(v), "launches": len(v)} for k, v in agg.items()}
    res["_source"] = rep
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
