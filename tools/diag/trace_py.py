import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1509_08197_b200 import engine as E
from paper_1509_08197_b200.synthetic import make_batch
sc = make_batch(2)
L = torch.from_numpy(np.stack([s.pair.left.data for s in sc])).cuda()
R = torch.from_numpy(np.stack([s.pair.right.data for s in sc])).cuda()
def T(label, fn):
    torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print(f"{label:20s} {1e3*(time.perf_counter()-t):8.3f} ms"); return r
for rep in range(3):
    print("rep", rep)
    il = T("to_f64", lambda: E.to_f64(L)); ir = E.to_f64(R)
    pl = T("prepare", lambda: E.prepare(il, False)[3]); pr = E.prepare(ir, False)[3]
    eu, ev, ew, key, nE = T("grid_edges", lambda: E.grid_edges(il))
    in_tree, comp, rounds = T("mst", lambda: E.mst(8 * 370 * 463, eu, ev, key))
    f = T("forest_create", lambda: E.DeviceForest(8 * 370 * 463, eu, ev, ew, in_tree, comp, 0.1))
    T("set_lanes", lambda: f.set_lanes_range(0, 81))
    lev = E.Level(0, 370, 463, 3, 80, il, ir, pl, pr)
    T("aggregate", lambda: f.aggregate(lev))
    T("pair_stats", lambda: E._per_pair_stats(f, 8, 370 * 463, 80))
    T("full baseline", lambda: E.run_baseline_batch(L, R, 80))
