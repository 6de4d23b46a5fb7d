"""Summarise an .ncu-rep (read here, no GPU needed) into a markdown table."""
import csv
import io
import subprocess
import sys

KEYS = [("time_us", "gpu__time_duration.sum", 1.0),
        ("dram_rd_MB", "dram__bytes_read.sum", 1.0), ("dram_wr_MB", "dram__bytes_write.sum", 1.0),
        ("dram_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
        ("tensor_%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
        ("l2_%", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
        ("issue_%", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
        ("warps_%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
        ("regs", "launch__registers_per_thread", 1.0),
        ("inst_M", "smsp__inst_executed.sum", 1e-6)]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6,
             "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}
    print("| kernel | " + " | ".join(k for k, _, _ in KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        vals = []
        for _, m, s in KEYS:
            v = d.get(m, "")
            try:
                x = float(v.replace(',', '')) * s * scale.get(units.get(m, ""), 1.0)
                vals.append(f"{x:.1f}")
            except ValueError:
                vals.append(v)
        print(f"| {d['Kernel Name'].split('(')[0][-40:]} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
