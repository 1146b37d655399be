"""Print source lines with the most warp-stall samples from an ncu report.
usage: python tools/ncu_source.py REPORT [min_pct] [ncu filter args...] (needs ncu on PATH)"""
import csv, io, subprocess, sys
rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
extra = sys.argv[3:]  # e.g. -k regex:NAME --launch-skip 2 --launch-count 1
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"] + extra,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
def num(x):
    try: return float(x)
    except ValueError: return 0.0
hdr = None; fn = ""
blocks = []
for r in rows:
    if r and r[0] == "Function Name": fn = r[1] if len(r) > 1 else ""
    if r and r[0] == "Line No":
        hdr = r; blocks.append((fn, hdr, [])); continue
    if hdr and blocks: blocks[-1][2].append(r)
for fn, hdr, data in blocks:
    if "Warp Stall Sampling (All Samples)" not in hdr: continue
    si = hdr.index("Warp Stall Sampling (All Samples)"); ie = hdr.index("Instructions Executed")
    tot = sum(num(r[si]) for r in data if len(r) > si and r[0])
    if tot == 0: continue
    print(f"== {fn[:90]}  samples={tot:.0f}")
    for r in data:
        if len(r) > si and r[0] and num(r[si]) >= thr / 100 * tot:
            print(f"{r[0]:>5} {100*num(r[si])/tot:5.1f}% inst={r[ie]:>10}  {r[1].strip()[:100]}")
