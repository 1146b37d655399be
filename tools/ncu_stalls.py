"""Stall-reason breakdown and top SASS instructions of one kernel launch.
usage: python tools/ncu_stalls.py REPORT [top] [ncu filter args...]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"] + sys.argv[3:],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hi = [k for k, x in enumerate(r) if x and x[0] == "Address"][0]
h = r[hi]
si = h.index("Warp Stall Sampling (All Samples)")
def num(v):
    try: return float(v)
    except ValueError: return 0.0
data = [x for x in r[hi + 1:] if len(x) == len(h)]
tot = sum(num(x[si]) for x in data) or 1
cols = [c for c in range(len(h)) if h[c].startswith("stall_") and "(Not" not in h[c]]
agg = {h[c]: sum(num(x[c]) for x in data) for c in cols}
print("stalls:", ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for k in sorted(range(len(data)), key=lambda k: -num(data[k][si]))[:top]:
    x = data[k]
    rs = sorted(((num(x[c]), h[c][6:]) for c in cols if num(x[c]) > 0), reverse=True)[:2]
    print(f"{k:5d} {100*num(x[si])/tot:5.1f}%  {x[1][:56]:56s} {rs}")
