"""Heavy-path length distribution of the MST forest of one config (pair 0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_08197_b200 import engine as E
from paper_1509_08197_b200.synthetic import make_batch, CONFIGS
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
spec = CONFIGS[cid]
sc = make_batch(cid, 1)
L = torch.from_numpy(np.stack([s.pair.left.data for s in sc])).cuda()
H, W = spec.height, spec.width
il = E.to_f64(L)
eu, ev, ew, key, nE = E.grid_edges(il)
in_tree, comp, rounds = E.mst(H * W, eu, ev, key)
f = E.DeviceForest(H * W, eu, ev, ew, in_tree, comp, 0.1)
ex = f.export()
parent = ex["parent"].cpu().numpy().astype(np.int64)
size = ex["size"].cpu().numpy().astype(np.int64)
n = parent.size
v = np.arange(n)
nonroot = parent != v
# heavy child: max size, ties -> lower id
order = np.lexsort((v[nonroot], -size[nonroot], parent[nonroot]))
ch = v[nonroot][order]; par = parent[nonroot][order]
first = np.ones(ch.size, bool); first[1:] = par[1:] != par[:-1]
heavy = np.full(n, -1); heavy[par[first]] = ch[first]
is_heavy = nonroot & (heavy[np.where(nonroot, parent, 0)] == v)
hp = np.where(is_heavy, parent, v)
while True:
    nx = hp[hp]
    if np.array_equal(nx, hp): break
    hp = nx
plen = np.bincount(hp, minlength=n)
heads = plen > 0
lens = plen[heads]
print(f"C{cid}: n={n} paths={lens.size} max_len={lens.max()}")
for lo, hi in [(1, 1), (2, 2), (3, 4), (5, 8), (9, 64), (65, 10**9)]:
    sel = (lens >= lo) & (lens <= hi)
    print(f"  len {lo:>4}-{hi:<10}: paths {sel.sum():>9} ({100*sel.mean():5.1f}%)  nodes {lens[sel].sum():>9} ({100*lens[sel].sum()/n:5.1f}%)")
nlc = np.bincount(parent[nonroot & ~is_heavy], minlength=n)
print(f"  nodes with light children: {100*(nlc>0).mean():.1f}%  light children total {nlc.sum()}")
