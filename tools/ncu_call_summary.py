"""Summary of ONE hdp_aggregate_wta call from an `ncu --page raw --csv`
export: the launches from a raw-cost pre-pass (k_ecost*) through the next
k_keys_finish.  Prints a per-launch table and writes the call's DRAM traffic
(the bench's roofline.traffic) as JSON.
usage: python tools/ncu_call_summary.py RAW.csv OUT.json LABEL"""
import csv
import json
import sys

raw, out_json, label = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(raw)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, units = rows[hi], rows[hi + 1]
data = rows[hi + 2:]
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0,
         "msecond": 1e3, "nsecond": 1e-3}


def val(r, col):
    i = h.index(col)
    return float(r[i].replace(",", "")) * scale.get(units[i], 1.0)


names = [r[h.index("Kernel Name")] for r in data]
start = next(i for i, n in enumerate(names) if "k_ecost" in n)
while start > 0 and "k_pack_rec8" in names[start - 1]:  # the byte-record pack passes belong to the call
    start -= 1
end = next(i for i in range(start, len(names)) if "k_keys_finish" in names[i])
call = data[start:end + 1]
tot_b = tot_t = 0.0
print(f"{'kernel':>16} {'grid':>8} {'us':>9} {'readMB':>9} {'writeMB':>9} {'dram%':>6} {'warps%':>6}")
for r in call:
    b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    t = val(r, "gpu__time_duration.sum")
    tot_b += b
    tot_t += t
    nm = r[h.index("Kernel Name")].split("(")[0].split("::")[-1].replace("void ", "")[:16]
    print(f"{nm:>16} {r[h.index('launch__grid_size')]:>8} {t:9.1f} {val(r, 'dram__bytes_read.sum')/1e6:9.1f} "
          f"{val(r, 'dram__bytes_write.sum')/1e6:9.1f} "
          f"{float(r[h.index('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')]):6.1f} "
          f"{float(r[h.index('sm__warps_active.avg.pct_of_peak_sustained_active')]):6.1f}")
print(f"call: {len(call)} launches, {tot_t:.1f} us serialised, DRAM {tot_b/1e9:.3f} GB "
      f"({tot_b/1e3/tot_t:.1f} GB/s over the serialised time)")
json.dump({"bytes_per_call": tot_b, "launches": len(call), "serialised_us": tot_t, "label": label,
           "source": "ncu --set full --clock-control none, dram__bytes_read.sum + dram__bytes_write.sum summed "
                     "over the launches of one hdp_aggregate_wta call (k_ecost* .. k_keys_finish)"},
          open(out_json, "w"), indent=1)
