"""Dense C2 pipeline time vs batch size (device events): how far the step is
from linear in the work (latency / launch bound vs bandwidth bound)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1509_08197_b200 import engine as E
from paper_1509_08197_b200.synthetic import make_batch, CONFIGS
sc = make_batch(2, 16)
Lh = np.stack([s.pair.left.data for s in sc]); Rh = np.stack([s.pair.right.data for s in sc])
for b in (1, 2, 4, 8, 16):
    L = torch.from_numpy(Lh[:b]).cuda(); R = torch.from_numpy(Rh[:b]).cuda()
    ms = []
    for it in range(8):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        agg = []
        torch.cuda.synchronize(); e0.record()
        E.run_baseline_fused(L, R, 80, agg_ms=agg)
        e1.record(); torch.cuda.synchronize()
        if it >= 3: ms.append((e0.elapsed_time(e1), agg[0]))
    t = np.median([m[0] for m in ms]); a = np.median([m[1] for m in ms])
    print(f"batch {b:2d}: step {t:7.3f} ms  agg {a:6.3f} ms  tree+rest {t-a:6.3f} ms  per pair {t/b:6.3f} ms")
