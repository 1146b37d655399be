"""Instructions executed per CUDA source line of one profiled kernel.
usage: python tools/ncu_lines.py REPORT [top]"""
import csv, subprocess, sys, io
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; data = []
for r in rows:
    if r and r[0] == "Line No": hdr = r; continue
    if hdr: data.append(r)
ie = hdr.index("Instructions Executed"); si = hdr.index("Warp Stall Sampling (All Samples)")
def num(x):
    try: return float(x)
    except ValueError: return 0.0
d = [r for r in data if len(r) > ie and r[0]]
tot = sum(num(r[ie]) for r in d); ts = sum(num(r[si]) for r in d) or 1
print(f"total warp-instructions {tot:.0f}")
for r in sorted(d, key=lambda r: -num(r[si]))[:top]:
    print(f"inst {100*num(r[ie])/tot:5.1f}%  stall {100*num(r[si])/ts:5.1f}%  {r[0]:>5} {r[1].strip()[:110]}")
