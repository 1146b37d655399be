"""Kernel-level view of the occasional slow C4 HDP step: profiles N reps (CUPTI),
then lists kernels that ran >= 50 ms longer than their name's median and GPU idle
gaps >= 50 ms (with the kernels around them).
usage: python tools/diag/c4_outliers.py [reps]"""
import os, sys, statistics
from collections import defaultdict
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
from paper_1509_08197_b200 import engine as E
from paper_1509_08197_b200.aggregation import SIZE_CLASS_PRESETS
from paper_1509_08197_b200.hdp_model import GmmModel
from torch.profiler import ProfilerActivity, profile
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
wl = bench.WORKLOADS["c4_hdp"]
spec, scenes = bench.scenes_for("c4_hdp", 0)
L = torch.from_numpy(np.stack([s.pair.left.data for s in scenes])).cuda()
R = torch.from_numpy(np.stack([s.pair.right.data for s in scenes])).cuda()
model = GmmModel.parse(bench.load_model_text())
pre = SIZE_CLASS_PRESETS[wl["size_class"]]
def step():
    E.run_hdp_batch(L, R, spec.d_max, model, levels=wl["levels"], delta0=pre["delta0"], beta=pre["beta"],
                    tree_kind=wl.get("tree", "mst"))
for _ in range(3):
    step()
torch.cuda.synchronize()
times = []
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for r in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); step(); e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
print("reps:", " ".join(f"{t:.0f}" for t in times))
evs = sorted((e for e in prof.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
by = defaultdict(list)
for e in evs:
    by[e.name[:60]].append((e.time_range.end - e.time_range.start) / 1e3)
med = {k: statistics.median(v) for k, v in by.items()}
t0 = evs[0].time_range.start
print("long kernels:")
for e in evs:
    d = (e.time_range.end - e.time_range.start) / 1e3
    if d - med[e.name[:60]] >= 50:
        print(f"  at {(e.time_range.start - t0) / 1e3:9.1f} ms: {d:8.1f} ms (median {med[e.name[:60]]:.1f})  {e.name[:70]}")
print("idle gaps:")
last_end, last = evs[0].time_range.end, evs[0]
for e in evs[1:]:
    gap = (e.time_range.start - last_end) / 1e3
    if gap >= 50:
        print(f"  at {(last_end - t0) / 1e3:9.1f} ms: {gap:8.1f} ms idle after {last.name[:40]} before {e.name[:40]}")
    if e.time_range.end > last_end:
        last_end, last = e.time_range.end, e
