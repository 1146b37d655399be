import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1509_08197_b200 import engine as E
from paper_1509_08197_b200.synthetic import make_batch
sc = make_batch(2)
L = torch.from_numpy(np.stack([s.pair.left.data for s in sc])).cuda()
R = torch.from_numpy(np.stack([s.pair.right.data for s in sc])).cuda()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    if rep == 2: os.environ["HDP_TRACE"] = "1"
    out = E.run_baseline_batch(L, R, 80, timing=True)
    torch.cuda.synchronize()
    print(f"rep {rep} total {1e3*(time.perf_counter()-t):.2f} ms", out.timings, file=sys.stderr)
