"""Per-kernel device time of one pipeline step (torch.profiler / CUPTI, not
serialised like ncu).  usage: python tools/kprof.py LEG [reps]
LEG: c5 | c2 | c2_hdp | c3_hdp | c4_hdp (bench.py workloads)."""
import os
import sys
from collections import defaultdict

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402
from paper_1509_08197_b200 import engine as E  # noqa: E402
from paper_1509_08197_b200.aggregation import SIZE_CLASS_PRESETS  # noqa: E402
from paper_1509_08197_b200.hdp_model import GmmModel  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_hdp"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
batch = int(sys.argv[3]) if len(sys.argv) > 3 else None
wl = bench.WORKLOADS[name]
spec, scenes = bench.scenes_for(name, 0, batch)
L = torch.from_numpy(np.stack([s.pair.left.data for s in scenes])).cuda()
R = torch.from_numpy(np.stack([s.pair.right.data for s in scenes])).cuda()
model = GmmModel.parse(bench.load_model_text())


def step():
    if wl["kind"] == "dense":
        E.run_baseline_fused(L, R, spec.d_max)
    else:
        pre = SIZE_CLASS_PRESETS[wl["size_class"]]
        E.run_hdp_batch(L, R, spec.d_max, model, levels=wl["levels"], delta0=pre["delta0"],
                        beta=pre["beta"], tree_kind=wl.get("tree", "mst"))


for _ in range(2):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    step()
e1.record()
torch.cuda.synchronize()
print(f"{name}: {e0.elapsed_time(e1) / reps:.2f} ms per step (events, no profiler)")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        step()
    torch.cuda.synchronize()
tot = defaultdict(float)
cnt = defaultdict(int)
for ev in prof.events():
    if ev.device_type.name == "CUDA":
        k = ev.name.split("(")[0][:70]
        tot[k] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        cnt[k] += 1
s = sum(tot.values())
print(f"kernel time sum {s / reps / 1e3:.2f} ms per step, {sum(cnt.values()) // reps} launches per step")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:40]:
    print(f"  {v / reps / 1e3:9.3f} ms {100 * v / s:5.1f}% {cnt[k] // reps:5d}  {k}")
if os.environ.get("KPROF_TIMELINE"):
    pat = os.environ["KPROF_TIMELINE"].split(",")
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    t0 = min(e.time_range.start for e in evs)
    print("timeline (ms from first kernel): start end dur name")
    for e in sorted(evs, key=lambda e: e.time_range.start):
        if any(p in e.name for p in pat):
            print(f"  {(e.time_range.start - t0) / 1e3:9.3f} {(e.time_range.end - t0) / 1e3:9.3f} "
                  f"{(e.time_range.end - e.time_range.start) / 1e3:8.3f}  {e.name[:60]}")
    print(f"  last kernel end {(max(e.time_range.end for e in evs) - t0) / 1e3:.3f}")
if os.environ.get("KPROF_LONG"):
    thr = float(os.environ["KPROF_LONG"])
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    t0 = min(e.time_range.start for e in evs)
    print(f"kernels longer than {thr} ms:")
    for e in sorted(evs, key=lambda e: e.time_range.start):
        d = (e.time_range.end - e.time_range.start) / 1e3
        if d >= thr:
            print(f"  {(e.time_range.start - t0) / 1e3:9.3f} {d:8.3f}  {e.name[:70]}")
