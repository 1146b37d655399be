"""Aggregation-call and step times of the dense pipeline (A/B of library
builds via HDP_LIB).  usage: python tools/agg_ab.py [reps] [legs]"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1509_08197_b200 import engine as E  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
legs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["c5", "c2"]
tag = os.path.basename(os.environ.get("HDP_LIB", "default"))
for name in legs:
    spec, scenes = bench.scenes_for(name, 0)
    L = torch.from_numpy(np.stack([s.pair.left.data for s in scenes])).cuda()
    R = torch.from_numpy(np.stack([s.pair.right.data for s in scenes])).cuda()
    ref = None
    for _ in range(2):
        ref = E.run_baseline_fused(L, R, spec.d_max)
    agg, step = [], []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = E.run_baseline_fused(L, R, spec.d_max, agg_ms=agg)
        e1.record()
        torch.cuda.synchronize()
        step.append(e0.elapsed_time(e1))
    same = bool(torch.equal(out.disparity, ref.disparity))
    print(f"{tag:>20} {name}: agg {statistics.median(agg):7.3f} ms  step {statistics.median(step):7.3f} ms"
          f"  (min agg {min(agg):.3f})  deterministic={same}", flush=True)
