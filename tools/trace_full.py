"""Repeat the dense pipeline on one config; with HDP_TRACE=1 the library
prints per-stage times (synchronising) to stderr."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_08197_b200 import engine as E
from paper_1509_08197_b200.synthetic import make_batch, CONFIGS
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
spec = CONFIGS[cid]
sc = make_batch(cid, 1) if cid == 5 else make_batch(cid)
L = torch.from_numpy(np.stack([s.pair.left.data for s in sc])).cuda()
R = torch.from_numpy(np.stack([s.pair.right.data for s in sc])).cuda()
for rep in range(reps):
    torch.cuda.synchronize(); t = time.perf_counter()
    E.run_baseline_batch(L, R, spec.d_max)
    torch.cuda.synchronize()
    print(f"rep {rep}: {1e3*(time.perf_counter()-t):8.3f} ms", file=sys.stderr, flush=True)
