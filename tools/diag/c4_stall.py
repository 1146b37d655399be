"""Where does an occasional slow C4 HDP step stall?  Host wall-clock between the
level callbacks (no extra syncs) of every rep; prints the per-level host times of
the reps that took more than 1.3x the median.
usage: python tools/diag/c4_stall.py [reps]"""
import os, sys, time, statistics
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
from paper_1509_08197_b200 import engine as E
from paper_1509_08197_b200.aggregation import SIZE_CLASS_PRESETS
from paper_1509_08197_b200.hdp_model import GmmModel
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 14
wl = bench.WORKLOADS["c4_hdp"]
spec, scenes = bench.scenes_for("c4_hdp", 0)
L = torch.from_numpy(np.stack([s.pair.left.data for s in scenes])).cuda()
R = torch.from_numpy(np.stack([s.pair.right.data for s in scenes])).cuda()
model = GmmModel.parse(bench.load_model_text())
pre = SIZE_CLASS_PRESETS[wl["size_class"]]
if os.environ.get("C4_RESERVE_GB"):
    from paper_1509_08197_b200 import _lib
    _lib.call("hdp_pool_reserve", int(float(os.environ["C4_RESERVE_GB"]) * 2**30), _lib.stream())
rows = []
for r in range(reps):
    torch.cuda.synchronize()
    marks = [("start", time.perf_counter())]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    E.run_hdp_batch(L, R, spec.d_max, model, levels=wl["levels"], delta0=pre["delta0"], beta=pre["beta"],
                    tree_kind=wl.get("tree", "mst"), on_level=lambda o: marks.append((f"L{o.level}", time.perf_counter())))
    marks.append(("queued", time.perf_counter()))
    e1.record()
    torch.cuda.synchronize()
    marks.append(("drained", time.perf_counter()))
    rows.append((e0.elapsed_time(e1), marks))
med = statistics.median(x[0] for x in rows)
print(f"median {med:.1f} ms; reps: " + " ".join(f"{x[0]:.0f}" for x in rows))
for i, (ms, marks) in enumerate(rows):
    if i == 3 or ms > 1.3 * med:
        print(f"rep {i} ({ms:.0f} ms) host ms between marks: " +
              " ".join(f"{b[0]}:{1e3 * (b[1] - a[1]):.0f}" for a, b in zip(marks, marks[1:])))
