"""Per-launch summary of an ncu --set full report.
usage: python tools/ncu_launches.py REPORT [name-regex]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
want = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"), ("launch__grid_size", "grid"),
        ("smsp__inst_executed.sum", "inst"), ("dram__bytes_read.sum", "rdMB"), ("dram__bytes_write.sum", "wrMB"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%")]
idx = [(h.index(c), n) for c, n in want if c in h]
units = r[1]
print("  ".join(f"{n:>10}" for _, n in idx))
for row in r[2:]:
    if pat and not pat.search(row[h.index("Kernel Name")]): continue
    vals = []
    for i, n in idx:
        v = row[i]
        if n == "kernel": v = v.split("(")[0][-14:]
        elif n in ("rdMB", "wrMB"):
            scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(units[i], 1.0)
            v = f"{float(v.replace(',', '')) * scale:.2f}"
        vals.append(f"{v:>10}")
    print("  ".join(vals))
