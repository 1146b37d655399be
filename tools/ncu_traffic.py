"""DRAM bytes (read + write) summed over the launches of an ncu report: the
`roofline.traffic` figure of one aggregation call.
usage: python tools/ncu_traffic.py REPORT"""
import csv, io, json, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, units = r[0], r[1]
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot = 0.0
names = set()
skip = ("k_light_depth", "k_light_steps")  # forest-build kernels the name regex also catches
for row in r[2:]:
    if any(k in row[h.index("Kernel Name")] for k in skip):
        continue
    for c in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(c)
        tot += float(row[i].replace(",", "")) * scale.get(units[i], 1.0)
    names.add(row[h.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0])
print(json.dumps({"bytes_per_call": tot,  "kernels": ", ".join(sorted(names)),
                  "source": "ncu --set full --clock-control none, dram__bytes_read.sum + dram__bytes_write.sum "
                            "summed over the launches of one hdp_aggregate_wta call (C2 dense, 8 pairs)"}, indent=1))
