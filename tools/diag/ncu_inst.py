"""Source lines of one kernel ranked by executed instructions (and stall samples).
usage: python tools/ncu_inst.py REPORT [top] [ncu filter args...]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"] + sys.argv[3:],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
def num(x):
    try: return float(x)
    except ValueError: return 0.0
hdr = None; data = []
for r in rows:
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and r and r[0] and len(r) == len(hdr): data.append(r)
ie = hdr.index("Instructions Executed"); si = hdr.index("Warp Stall Sampling (All Samples)")
agg = {}
for r in data:
    k = (r[0], r[1].strip()[:90])
    a = agg.setdefault(k, [0.0, 0.0]); a[0] += num(r[ie]); a[1] += num(r[si])
ti = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {ti:.0f}")
for (ln, src), (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln:>5} {i:10.0f} {100*i/ti:5.1f}%  stall {100*s/ts:5.1f}%  {src}")
