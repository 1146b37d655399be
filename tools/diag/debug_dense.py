import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1509_08197_b200 import engine as E
from oracle import oracle as O
g = np.load("tests/golden/pipelines.npz")
L = torch.from_numpy(g["c1_left"][None]).cuda(); R = torch.from_numpy(g["c1_right"][None]).cuda()
out = E.run_baseline_batch(L, R, 16, want_volume=True, keep_forest=True)
vol = out.extra["volume"].cpu().numpy()
ref = O.run_baseline(g["c1_left"], g["c1_right"], 16)
d2, b2, s2, rvol, roff = O._layer_wta(g["c1_left"].astype(np.float64), g["c1_right"].astype(np.float64), 16, ref.forest, 0.1, want_volume=True)
gv = vol[: rvol.size].reshape(-1, 17); rv = rvol.reshape(-1, 17)
err = np.abs(gv - rv) / (np.abs(rv) + 1e-7)
bad = np.flatnonzero(err.max(1) > 1e-3)
print("volume bad nodes", bad.size, "of", gv.shape[0], bad[:10])
disp = out.disparity[0].cpu().numpy().ravel()
print("disp mismatches", (disp != ref.disparity.ravel()).sum())
vd = gv.argmin(1)
print("argmin of gpu volume vs gpu disp mismatch", (vd != disp).sum())
f = out.forest
o = {k: v.cpu().numpy() for k, v in f.export().items()}
print("phases", f.n_phases, "paths", f.n_paths)
if bad.size:
    i = bad[0]; print("node", i, "gpu", gv[i][:6], "ref", rv[i][:6], "parent", o["parent"][i], "depth", o["depth"][i])
wrong = np.flatnonzero(disp != vd)
# classify by path length: recompute heavy-path membership from parent/size
par = o["parent"]; size = o["size"]; n = par.size
heavy = np.full(n, -1)
for v in range(n):
    p = par[v]
    if p != v and (heavy[p] < 0 or size[v] > size[heavy[p]] or (size[v] == size[heavy[p]] and v < heavy[p])):
        heavy[p] = v
is_head = np.array([par[v] == v or heavy[par[v]] != v for v in range(n)])
head = np.arange(n)
for v in range(n):
    h = v
    while not is_head[h]: h = par[h]
    head[v] = h
plen = np.bincount(head, minlength=n)
print("wrong nodes path-length histogram", np.bincount(np.minimum(plen[head[wrong]], 20)))
print("all nodes path-length hist", np.bincount(np.minimum(plen[head], 20)))
print("example wrong", wrong[:5], "gpu disp", disp[wrong[:5]], "argmin", vd[wrong[:5]])
