"""C5 dense: one-call pipeline vs step-by-step path, several reps (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1509_08197_b200 import engine as E
from paper_1509_08197_b200.synthetic import make_batch, CONFIGS
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
spec = CONFIGS[cid]
sc = make_batch(cid, 1) if cid == 5 else make_batch(cid)
L = torch.from_numpy(np.stack([s.pair.left.data for s in sc])).cuda()
R = torch.from_numpy(np.stack([s.pair.right.data for s in sc])).cuda()
for name, fn in [("fused", lambda: E.run_baseline_fused(L, R, spec.d_max)),
                 ("steps", lambda: E.run_baseline_batch(L, R, spec.d_max, timing=True)),
                 ("fused", lambda: E.run_baseline_fused(L, R, spec.d_max))]:
    for r in range(3):
        torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize()
        print(f"{name} rep{r}: {1e3*(time.perf_counter()-t):8.2f} ms", flush=True)
