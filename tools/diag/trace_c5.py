import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1509_08197_b200 import engine as E
from paper_1509_08197_b200.synthetic import make_batch, CONFIGS
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
spec = CONFIGS[cid]
sc = make_batch(cid, 1)
L = torch.from_numpy(np.stack([s.pair.left.data for s in sc])).cuda()
R = torch.from_numpy(np.stack([s.pair.right.data for s in sc])).cuda()
def T(label, fn):
    torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print(f"{label:20s} {1e3*(time.perf_counter()-t):8.3f} ms", flush=True); return r
H, W, d = spec.height, spec.width, spec.d_max
for rep in range(3):
    print("rep", rep)
    il = E.to_f64(L); ir = E.to_f64(R)
    pl = E.prepare(il, False)[3]; pr = E.prepare(ir, False)[3]
    eu, ev, ew, key, nE = T("grid_edges", lambda: E.grid_edges(il))
    in_tree, comp, rounds = T("mst", lambda: E.mst(H * W, eu, ev, key))
    f = T("forest_create", lambda: E.DeviceForest(H * W, eu, ev, ew, in_tree, comp, 0.1))
    T("set_lanes", lambda: f.set_lanes_range(0, d + 1))
    lev = E.Level(0, H, W, 3, d, il, ir, pl, pr)
    T("aggregate", lambda: f.aggregate(lev))
    del f
    T("full baseline", lambda: E.run_baseline_batch(L, R, d))
    pass
