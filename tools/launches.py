"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.
usage: python tools/launches.py FILE [--last-frac 0.5] [--top 25] [--per-launch PATTERN]"""
import csv, collections, sys, argparse
ap = argparse.ArgumentParser()
ap.add_argument("file")
ap.add_argument("--last-frac", type=float, default=0.5)
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--per-launch", default=None)
a = ap.parse_args()
rows = list(csv.reader(open(a.file)))
hdr = None; data = []
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
part = data[int(len(data) * (1 - a.last_frac)):]
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
agg = collections.OrderedDict()
for d in part:
    v = float(d["Metric Value"]) * scale[d["Metric Unit"]]
    name = d["Kernel Name"].split("(")[0][:70]
    x = agg.setdefault(name, [0, 0.0]); x[0] += 1; x[1] += v
    if a.per_launch and a.per_launch in name:
        print(f"   {name[:30]} grid={d['Grid Size']} {v:.1f} us")
tot = sum(v[1] for v in agg.values())
print(f"launches {len(part)}  total {tot:.1f} us")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:a.top]:
    print(f"{v[1]:10.1f} us {100*v[1]/tot:5.1f}% {v[0]:5d}  {k}")
