"""Host-side cost of the reference-signature API (run_baseline_pipeline_batch)
at C5 and C2: wall time of each stage of one call, after warm-up.
usage: python tools/api_prof.py"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1509_08197_b200 import aggregation as A  # noqa: E402
from paper_1509_08197_b200 import engine as E  # noqa: E402
from paper_1509_08197_b200.synthetic import CONFIGS, make_scene  # noqa: E402

for cid, b in ((5, 1), (2, 8)):
    spec = CONFIGS[cid]
    pairs = [make_scene(spec, i).pair for i in range(b)]
    for _ in range(3):
        A.run_baseline_pipeline_batch(pairs)
    torch.cuda.synchronize()
    for rep in range(3):
        t = [time.perf_counter()]
        ld, rd, ready = E.stage_pairs([p.left.data for p in pairs], [p.right.data for p in pairs])
        t.append(time.perf_counter())
        out = E.run_baseline_fused(ld, rd, spec.d_max, right_ready=ready, timing=True)
        t.append(time.perf_counter())
        d = out.disparity.cpu().numpy()
        t.append(time.perf_counter())
        c = out.min_cost.cpu().numpy().astype(np.float64)
        t.append(time.perf_counter())
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A.run_baseline_pipeline_batch(pairs)
        t1 = time.perf_counter()
        print(f"C{cid}: stage {1e3*(t[1]-t[0]):.2f} pipeline {1e3*(t[2]-t[1]):.2f} d2h disp {1e3*(t[3]-t[2]):.2f} "
              f"d2h cost+f64 {1e3*(t[4]-t[3]):.2f} | full API call {1e3*(t1-t0):.2f} ms", flush=True)
